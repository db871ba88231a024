"""Fine solvers F_n, F_n', F_n'^* and offsets b_n -- TEST INFRASTRUCTURE ONLY.

Paper: the fine solver is backward Euler with equidistant steps;
F_n is affine, F_n v = F_n' v + b_n with b_n := F_n 0 (eq.
F_n_affine); the adjoint F_n'^* is defined by (F_n'^* w, v) = (w, F_n' v)
(P:271-273), which for a product of m step solves is the product of the
transposed solves in reverse order.

One step of interval n (1-based), j = 1..m, global index g = (n-1)*m + j:
        (I + dt A) u_j = u_{j-1} + dt f(t_g)            (reading Z3)

1D: each step is one Thomas solve (oracle/csrc/oracle_thomas.c), pivots from
    the exact row sums of I + dt A (reading R-ACC).
2D, "oracle A" (fine_2d_banded): each step is one banded Cholesky solve of the
    5-point system (oracle/csrc/oracle_band.c) -- no sine basis.  Used to
    cross-validate oracle B below (tests/test_oracle_fine2d_banded.py).
2D, "oracle B" (fine_2d): A = T(x)I + I(x)T (5-point, Dirichlet).  The step is solved exactly by
    the classical fast-Poisson partial diagonalisation: transform the x index
    with the orthogonal sine matrix S (T = S diag(lam) S), then for every
    x-mode i solve the tridiagonal system ((1 + dt lam_i) I + dt T) in y with
    Thomas.  The state stays x-transformed across the m steps of one call
    (every step is still one exact linear solve); input and output are
    physical-space vectors.  Pinned against a dense direct solve.
"""
from __future__ import annotations

import numpy as np

from ._clib import band_factor, band_solve, thomas_batch


# --------------------------------------------------------------------- 1D
class Op1D:
    """A = tridiag(sub, diag, sup) on n interior points, time step dt, m steps.

    rowsum/colsum: exact row/column sums of A (problem data); when given, the
    Thomas pivots use the row-sum recurrence (oracle_thomas.c, reading R-ACC)."""

    def __init__(self, sub, diag, sup, dt: float, m: int, rowsum=None, colsum=None):
        self.n = len(diag)
        self.A = (np.asarray(sub, float), np.asarray(diag, float), np.asarray(sup, float))
        self.dt, self.m = float(dt), int(m)
        a, d, c = self.A
        # I + dt A, and its row sums 1 + dt * rowsum(A)
        self.T = (dt * a, 1.0 + dt * d, dt * c)
        self.T_rs = None if rowsum is None else 1.0 + dt * np.asarray(rowsum, float)
        # (I + dt A)^T: T^T[i, i-1] = T[i-1, i]; its row sums are T's column sums
        subT = np.zeros(self.n)
        supT = np.zeros(self.n)
        subT[1:] = self.T[2][:-1]
        supT[:-1] = self.T[0][1:]
        self.TT = (subT, self.T[1], supT)
        self.TT_rs = None if colsum is None else 1.0 + dt * np.asarray(colsum, float)

    def dense_A(self) -> np.ndarray:
        a, d, c = self.A
        return np.diag(d) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)


def fine_1d(op: Op1D, interval: int, X: np.ndarray, mode: str = "linear", src=None,
            src_index=None) -> np.ndarray:
    """Apply F_n (mode 'affine'), F_n' ('linear') or F_n'^* ('adjoint') to rows of X.

    X: (nvec, n).  src = (space[R, n], time[R, N*m], amp[nsrc, R]); src_index[v]
    selects the source of vector v (default 0).  Returns a new array.
    """
    X = np.array(X, dtype=np.float64, order="C", copy=True)
    if X.ndim == 1:
        return fine_1d(op, interval, X[None, :], mode, src, src_index)[0]
    nvec = X.shape[0]
    if mode == "adjoint":
        # transposed solves in reverse step order (all steps share A here, so the
        # reversal only matters formally; no source term in F'^*).
        for _ in range(op.m):
            thomas_batch(*op.TT, X, rowsum=op.TT_rs)
        return X
    for j in range(1, op.m + 1):
        if mode == "affine" and src is not None:
            space, time, amp = src
            g = (interval - 1) * op.m + j
            idx = np.zeros(nvec, dtype=int) if src_index is None else np.asarray(src_index)
            coef = amp[idx] * time[:, g - 1][None, :]          # (nvec, R)
            X += op.dt * (coef @ space)                          # f(x_i, t_g)
        thomas_batch(*op.T, X, rowsum=op.T_rs)
    return X


# --------------------------------------------------------------------- 2D
def sine_matrix(n: int) -> np.ndarray:
    """Orthogonal symmetric S_ij = sqrt(2/(n+1)) sin((i+1)(j+1) pi/(n+1))."""
    i = np.arange(1, n + 1, dtype=np.float64)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.outer(i, i) * np.pi / (n + 1))


class Op2D:
    """A = T(x)I + I(x)T with T = tridiag(sub, diag, sup) (constant coefficients)."""

    def __init__(self, sub, diag, sup, dt: float, m: int, rowsum=None):
        self.n = len(diag)
        n = self.n
        self.A1 = (np.asarray(sub, float), np.asarray(diag, float), np.asarray(sup, float))
        self.dt, self.m = float(dt), int(m)
        a, d, c = self.A1
        # eigenpairs of the constant-coefficient T: T = S diag(lam) S
        assert np.allclose(a[1:], a[1]) and np.allclose(d, d[0]) and np.allclose(c[:-1], c[0])
        self.S = sine_matrix(n)
        i = np.arange(1, n + 1, dtype=np.float64)
        # lam_i = d + 2c cos(i pi/(n+1)) = -4c sin^2(i pi / (2(n+1))) (d = -2c), no cancellation
        assert np.allclose(d[0], -2.0 * c[0])
        self.lam = -4.0 * c[0] * np.sin(i * np.pi / (2.0 * (n + 1))) ** 2
        self.Ty = (dt * a, 1.0 + dt * d, dt * c)   # I + dt T  (the y-direction part)
        # row sums of the line systems (1 + dt lam_i) I + dt T: 1 + dt rowsum(T), + shift
        self.Ty_rs = None if rowsum is None else 1.0 + dt * np.asarray(rowsum, float)

    def dense_A(self) -> np.ndarray:
        a, d, c = self.A1
        T = np.diag(d) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
        I = np.eye(self.n)
        return np.kron(T, I) + np.kron(I, T)


def fine_2d(op: Op2D, interval: int, X: np.ndarray, mode: str = "linear", src=None) -> np.ndarray:
    """X: (nvec, n, n) [vector, x-index, y-index].  A is symmetric and time
    independent, so F'^* = F' (mode 'adjoint' == 'linear').  src = (gx, gy)."""
    X = np.array(X, dtype=np.float64, copy=True)
    if X.ndim == 2:
        return fine_2d(op, interval, X[None], mode, src)[0]
    nvec, n = X.shape[0], op.n
    S = op.S
    V = np.ascontiguousarray(np.matmul(S, X))                     # x-transform: S along the x index
    shift = np.tile(op.dt * op.lam, nvec)
    for j in range(1, op.m + 1):
        if mode == "affine" and src is not None:
            gx, gy = src
            g = (interval - 1) * op.m + j
            Sg = S @ gx[:, g - 1, :].T                                 # (n, nb)
            V += op.dt * (Sg @ gy[:, g - 1, :])[None]                  # S f_g
        thomas_batch(*op.Ty, V.reshape(nvec * n, n), shift, rowsum=op.Ty_rs)
    return np.matmul(S, V)


class Op2DBanded:
    """Oracle A: the n x n 5-point Dirichlet Laplacian with unit diffusion
    (BJ C3/C5), I + dt A factored once by banded Cholesky."""

    def __init__(self, n: int, dt: float, m: int):
        self.n, self.dt, self.m = int(n), float(dt), int(m)
        self.L = band_factor(self.n, self.dt)


def fine_2d_banded(op: Op2DBanded, interval: int, X: np.ndarray, mode: str = "linear",
                   src=None) -> np.ndarray:
    """As fine_2d, by m banded solves per call (X: (nvec, n, n) [x, y]).  A is
    symmetric and time independent, so the adjoint is the same product."""
    X = np.array(X, dtype=np.float64, copy=True)
    if X.ndim == 2:
        return fine_2d_banded(op, interval, X[None], mode, src)[0]
    nvec, n = X.shape[0], op.n
    V = np.ascontiguousarray(X.reshape(nvec, n * n))
    for j in range(1, op.m + 1):
        if mode == "affine" and src is not None:
            gx, gy = src
            g = (interval - 1) * op.m + j
            f = gx[:, g - 1, :].T @ gy[:, g - 1, :]              # f[ix, iy] = sum_b gx gy
            V += op.dt * f.reshape(1, n * n)
        band_solve(n, op.L, V)
    return V.reshape(nvec, n, n)


class DenseOp:
    """A linear F' given by its matrix (tests only: operators with a prescribed
    SVD for the rSVD pins).  mode 'linear' applies F, 'adjoint' F^T."""

    def __init__(self, F: np.ndarray):
        self.F = np.asarray(F, dtype=np.float64)
        self.n = self.F.shape[0]


# ------------------------------------------------- time-dependent pencils
class OpPencil:
    """Time-dependent 1D pencil (Exp 2): step
    g (global, 1-based) solves (M + dt A(t_g)) u_g = M u_{g-1} + dt l(t_g)
    with its own tridiagonal L_g = M + dt A(t_g).  L: (sub, diag, sup) arrays
    of shape (nsteps, n); rowsum: exact row sums of L_g (nsteps, n) or None;
    M: (sub, diag, sup) of length n, or None for M = I."""

    def __init__(self, L, dt: float, m: int, rowsum=None, M=None):
        self.L = tuple(np.asarray(a, float) for a in L)
        self.nsteps, self.n = self.L[1].shape
        self.dt, self.m = float(dt), int(m)
        self.rowsum = None if rowsum is None else np.asarray(rowsum, float)
        self.M = None if M is None else tuple(np.asarray(a, float) for a in M)


def _tridiag_apply(T, X, transpose=False):
    """rows of X times the tridiagonal T = (sub, diag, sup) (or its transpose)."""
    sub, diag, sup = T
    Y = X * diag
    if not transpose:
        Y[:, 1:] += X[:, :-1] * sub[1:]          # T[i, i-1] x_{i-1}
        Y[:, :-1] += X[:, 1:] * sup[:-1]         # T[i, i+1] x_{i+1}
    else:
        Y[:, 1:] += X[:, :-1] * sup[:-1]         # T^T[i, i-1] = T[i-1, i]
        Y[:, :-1] += X[:, 1:] * sub[1:]          # T^T[i, i+1] = T[i+1, i]
    return Y


def fine_pencil(op: OpPencil, interval: int, X: np.ndarray, mode: str = "linear", src=None,
                src_index=None) -> np.ndarray:
    """F_n (affine), F_n' (linear) or F_n'^T (adjoint, Euclidean transpose of the
    product: the transposed steps in reverse order, each followed by M^T)."""
    X = np.array(X, dtype=np.float64, order="C", copy=True)
    if X.ndim == 1:
        return fine_pencil(op, interval, X[None, :], mode, src, src_index)[0]
    nvec = X.shape[0]
    g0 = (interval - 1) * op.m
    assert g0 + op.m <= op.nsteps, "interval beyond the operator's steps"
    if mode == "adjoint":
        for j in range(op.m, 0, -1):
            g = g0 + j
            a, d, c = (arr[g - 1] for arr in op.L)
            aT = np.zeros_like(a)
            cT = np.zeros_like(c)
            aT[1:] = c[:-1]                      # L^T[i, i-1] = L[i-1, i]
            cT[:-1] = a[1:]                      # L^T[i, i+1] = L[i+1, i]
            thomas_batch(aT, d, cT, X)
            if op.M is not None:
                X = np.ascontiguousarray(_tridiag_apply(op.M, X, transpose=True))
        return X
    for j in range(1, op.m + 1):
        g = g0 + j
        if op.M is not None:
            X = np.ascontiguousarray(_tridiag_apply(op.M, X))
        if mode == "affine" and src is not None:
            space, time, amp = src
            idx = np.zeros(nvec, dtype=int) if src_index is None else np.asarray(src_index)
            coef = amp[idx] * time[:, g - 1][None, :]
            X += op.dt * (coef @ space)
        a, d, c = (arr[g - 1] for arr in op.L)
        thomas_batch(a, d, c, X, rowsum=None if op.rowsum is None else op.rowsum[g - 1])
    return X


def dense_step_product(op: OpPencil, interval: int) -> np.ndarray:
    """F_n' as the dense product of its steps, (L_g^{-1} M) for g in the interval
    (brute force for tiny n; a pin for fine_pencil)."""
    n = op.n
    F = np.eye(n)
    Md = np.eye(n) if op.M is None else (np.diag(op.M[1]) + np.diag(op.M[0][1:], -1) + np.diag(op.M[2][:-1], 1))
    for j in range(1, op.m + 1):
        g = (interval - 1) * op.m + j
        a, d, c = (arr[g - 1] for arr in op.L)
        Lg = np.diag(d) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
        F = np.linalg.solve(Lg, Md @ F)
    return F


# ---------------------------------------------------------------- dispatch
def make_op(cfg):
    from workloads import generators as G
    if cfg.problem.startswith("exp2"):
        from workloads import exp2
        L, rs, M = exp2.step_matrices(cfg.problem, cfg.n, cfg.T, cfg.N * cfg.m)
        return OpPencil(L, cfg.dt, cfg.m, rowsum=rs, M=M)
    if cfg.dim == 1:
        rs, cs = G.operator_1d_sums(cfg)
        return Op1D(*G.operator_1d(cfg), cfg.dt, cfg.m, rowsum=rs, colsum=cs)
    return Op2D(*G.laplacian_1d_for_2d(cfg), cfg.dt, cfg.m,
                rowsum=G.laplacian_1d_for_2d_sums(cfg))


def fine(op, interval, X, mode="linear", src=None, src_index=None):
    if isinstance(op, DenseOp):
        X = np.asarray(X, dtype=np.float64)
        return X @ (op.F if mode == "adjoint" else op.F.T)
    if isinstance(op, Op1D):
        return fine_1d(op, interval, X, mode, src, src_index)
    if isinstance(op, OpPencil):
        return fine_pencil(op, interval, X, mode, src, src_index)
    return fine_2d(op, interval, X, mode, src)


def fine_trajectory(op, interval, X, src=None, src_index=None):
    """[x_0, x_1, ..., x_m]: the affine fine trajectory of interval `interval`
    from X, one step at a time (Op1D / OpPencil)."""
    X = np.array(X, dtype=np.float64)
    out = [X.copy()]
    if isinstance(op, Op1D):
        one = Op1D.__new__(Op1D)
        one.__dict__.update(op.__dict__)
        one.m = 1
        for j in range(1, op.m + 1):
            g = (interval - 1) * op.m + j        # global step of step j
            X = fine_1d(one, g, X, "affine", src, src_index) if src is not None else fine_1d(one, g, X, "linear")
            out.append(X.copy())
        return out
    if isinstance(op, OpPencil):
        one = OpPencil.__new__(OpPencil)
        one.__dict__.update(op.__dict__)
        one.m = 1
        for j in range(1, op.m + 1):
            g = (interval - 1) * op.m + j
            X = fine_pencil(one, g, X, "affine" if src is not None else "linear", src, src_index)
            out.append(X.copy())
        return out
    raise TypeError("fine_trajectory: 1D operators only")


def sequential_reference(op, u0, N: int, src=None, src_index=None):
    """u_{n+1} = F_{n+1} u_n, 0 <= n < N.  u0: (nvec, ...) batch."""
    out = [np.array(u0, dtype=np.float64)]
    for n in range(1, N + 1):
        out.append(fine(op, n, out[-1], "affine", src, src_index))
    return np.stack(out)
