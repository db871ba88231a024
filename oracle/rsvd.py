"""Randomized SVD of the transfer operator F_n' -- TEST INFRASTRUCTURE ONLY.

Follows P:258-299 ("Computation of G_n", steps 1-6) in the paper's order:

 1. draw l = R_n + p random vectors omega_i (oracle/rng.py) and compute
    F_n' omega_i;
 2. orthonormal basis w_1..w_l of W = span{F_n' omega_i};
 3. compute F_n'^* w_i;
 4. orthonormal basis v_1..v_l of span{F_n'^* w_i};
 5. M_ij := (F_n'^* w_i, v_j), its SVD M = Psi Sigma Phi^T, and
    psi_r = sum_i Psi_{i,r} w_i,  phi_r = sum_i Phi_{i,r} v_i
    -- the paper's P:293-294 prints w and v the other way round; the printed
    assignment does not give the SVD of P_W F_n' (SURVEY finding 4, pinned
    in tests by ||F' - G'|| = sigma_{k+1}); reading Z5;
 6. return the first R_n triples.

Spectral coarse solver (eq. spectral_G):
    G_n v = sum_{r <= R_n} psi_r sigma_r (phi_r, v) + b_n.
Euclidean inner product throughout (V = R^m case; reading Z1).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fine import DenseOp, Op1D, OpPencil, fine
from .linalg import householder_qr, jacobi_svd, weighted_gram_schmidt
from .rng import gaussian_sketch


@dataclass
class Truncated:
    U: np.ndarray       # (n_dof, k)  left singular vectors psi_r
    sigma: np.ndarray   # (l,)        all computed singular values of P_W F_n'
    V: np.ndarray       # (n_dof, k)  right singular vectors phi_r
    k: int

    def apply_linear(self, X: np.ndarray) -> np.ndarray:
        """G_n' x for rows x of X (n_vec, n_dof)."""
        s = self.sigma[: self.k]
        return ((X @ self.V) * s) @ self.U.T


def _as_vectors(op, cols: np.ndarray) -> np.ndarray:
    """(n_dof, l) column block -> fine-solver batch layout."""
    if isinstance(op, (Op1D, OpPencil, DenseOp)):
        return np.ascontiguousarray(cols.T)
    n = op.n
    return np.ascontiguousarray(cols.T.reshape(-1, n, n))


def _as_columns(op, vecs: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(vecs.reshape(vecs.shape[0], -1).T)


def rsvd_interval(op, interval: int, k: int, p: int, seed: int, power_iterations: int = 0,
                  independent_adjoint: bool = False, inner=None) -> Truncated:
    """Steps 1-6 for the 1-based interval n = `interval`.

    power_iterations q: W = span{(F' F'^*)^q F' omega_i}, evaluated
    with an orthonormalisation (Householder) between the applications -- the
    same span in exact arithmetic (reading R-POW).
    independent_adjoint: step 3 applies F'^* to an independent
    Gaussian set Psi (stream 2) instead of the w_i; with Z = F'^* Psi and
    V = orth(Z), F' is approximated by W C V^T where C solves the two-sided
    sketch equation Psi^T W C = Psi^T F' V = Z^T V (Martinsson & Tropp's
    reconstruction, reading R-IND), and C replaces M of step 5."""
    l = k + p
    n_dof = op.n if isinstance(op, (Op1D, OpPencil)) else (op.F.shape[0] if isinstance(op, DenseOp) else op.n * op.n)
    if inner is not None:
        assert power_iterations == 0 and not independent_adjoint
        return _rsvd_weighted(op, interval, k, l, seed, inner, n_dof)
    # step 1
    Omega = gaussian_sketch(seed, interval - 1, n_dof, l)
    Y = _as_columns(op, fine(op, interval, _as_vectors(op, Omega), "linear"))
    for _ in range(power_iterations):
        Qy, _ = householder_qr(Y)
        Qz, _ = householder_qr(_as_columns(op, fine(op, interval, _as_vectors(op, Qy), "adjoint")))
        Y = _as_columns(op, fine(op, interval, _as_vectors(op, Qz), "linear"))
    # step 2
    W, _ = householder_qr(Y)
    if not independent_adjoint:
        # step 3
        Z = _as_columns(op, fine(op, interval, _as_vectors(op, W), "adjoint"))
        # step 4
        Vb, _ = householder_qr(Z)
        # step 5: M_ij = (F'^* w_i, v_j)
        M = Z.T @ Vb
    else:
        Psi = gaussian_sketch(seed, interval - 1, n_dof, l, stream=2)
        Z = _as_columns(op, fine(op, interval, _as_vectors(op, Psi), "adjoint"))
        Vb, _ = householder_qr(Z)
        M = np.linalg.solve(Psi.T @ W, Z.T @ Vb)
    Psi_, sig, Phi = jacobi_svd(M)
    U = W @ Psi_[:, :k]
    V = Vb @ Phi[:, :k]
    # step 6
    return Truncated(U=U, sigma=sig, V=V, k=k)


def _rsvd_weighted(op, interval, k, l, seed, inner, n_dof) -> Truncated:
    """Steps 1-6 with (.,.)_V = (.,.)_M, M = inner (tridiagonal (sub, diag, sup);
    the generalized SVD of eq. svd).  The V-adjoint is
    F'^* = M^{-1} F'^T M ((F'^* w, v)_M = (w, F' v)_M).  The basis of the
    Gram-Schmidt steps 2 and 4 is M-orthonormal; M_ij = (F'^* w_i, v_j)_M.
    The returned V holds M phi_r, so that apply_linear(x) = sum psi sigma (phi, x)_M.
    Test vectors: standard Gaussian in V, i.e. with E[(omega, v)_M^2] = ||v||_M^2:
    omega = C^{-1} xi, xi ~ N(0, I) (the seeded Philox draws), M = C^T C
    (reading R-WIP; the Cholesky factor is a library routine here).  The same
    seed then gives the same test vectors as the GPU's weighted view."""
    from .fine import _tridiag_apply
    ms, md, mp = (np.asarray(a, float) for a in inner)
    Mx = lambda X: _tridiag_apply((ms, md, mp), X.T).T          # columns
    Mfull = np.diag(md) + np.diag(ms[1:], -1) + np.diag(mp[:-1], 1)
    Cup = np.linalg.cholesky(Mfull).T                           # M = C^T C (library routine)
    Omega = np.linalg.solve(Cup, gaussian_sketch(seed, interval - 1, n_dof, l))
    Y = _as_columns(op, fine(op, interval, _as_vectors(op, Omega), "linear"))
    W = weighted_gram_schmidt(Y, Mx)
    FtMW = _as_columns(op, fine(op, interval, _as_vectors(op, Mx(W)), "adjoint"))   # F'^T M W
    Z = np.linalg.solve(Mfull, FtMW)                             # F'^* W
    Vb = weighted_gram_schmidt(Z, Mx)
    Mm = Z.T @ Mx(Vb)                                            # (F'^* w_i, v_j)_M
    Psi_, sig, Phi = jacobi_svd(Mm)
    U = W @ Psi_[:, :k]
    V = Vb @ Phi[:, :k]
    return Truncated(U=U, sigma=sig, V=Mx(V), k=k)


def exact_truncated(Fdense: np.ndarray, k: int) -> Truncated:
    """Truncated SVD of a dense F' (tiny grids only): eq. svd / spectral_G."""
    from .linalg import jacobi_svd as _svd
    Uf, s, Vf = _svd(Fdense)
    return Truncated(U=Uf[:, :k], sigma=s, V=Vf[:, :k], k=k)


def dense_transfer(op, interval: int = 1, mode: str = "linear") -> np.ndarray:
    """Matrix of F_n' by applying it to every unit vector (tiny grids only)."""
    n_dof = op.n if isinstance(op, (Op1D, OpPencil)) else (op.F.shape[0] if isinstance(op, DenseOp) else op.n * op.n)
    E = np.eye(n_dof)
    return _as_columns(op, fine(op, interval, _as_vectors(op, E), mode))


def delta_eps(truncs) -> tuple:
    """delta := max_n sigma_{n,1}, eps := max_n sigma_{n,R_n+1} (P:407-411,
    with the computed sigma_{n,k+1} as the estimate; Z19)."""
    delta = max(t.sigma[0] for t in truncs)
    eps = max(t.sigma[t.k] if t.k < len(t.sigma) else 0.0 for t in truncs)
    return delta, eps


def coarse_error_estimate(op, trunc: Truncated, interval: int, r: int, seed: int) -> float:
    """The failure-probability estimator of an adaptive p (Halko,
    Martinsson & Tropp 2011, Lemma 4.1): 10 sqrt(2/pi) max_{i<=r} ||(F' - G') omega_i||,
    omega_i i.i.d. N(0,1) (Philox counter word 3 = 3)."""
    n_dof = op.n if isinstance(op, (Op1D, OpPencil)) else (op.F.shape[0] if isinstance(op, DenseOp) else op.n * op.n)
    Om = gaussian_sketch(seed, interval - 1, n_dof, r, stream=3)
    FO = _as_columns(op, fine(op, interval, _as_vectors(op, Om), "linear"))
    GO = trunc.apply_linear(Om.T).T
    return 10.0 * np.sqrt(2.0 / np.pi) * float(np.max(np.linalg.norm(FO - GO, axis=0)))
