"""Dense linear algebra of the rSVD -- TEST INFRASTRUCTURE ONLY.

* householder_qr: orthonormal basis of span{columns} for rSVD steps 2 and 4
  (P:269-270).  The paper suggests modified Gram-Schmidt; the
  oracle uses Householder reflections (Golub & Van Loan, Alg. 5.2.1), which is
  unconditionally stable on the numerically rank-deficient snapshot blocks
  (SURVEY §0 finding 6).  No column dropping: l stays fixed (reading Z7).
* weighted_gram_schmidt: the same basis in the inner product (u, v)_M =
  u^T M v of V: classical Gram-Schmidt with one full
  reorthogonalisation pass (CGS2), every inner product and norm in M.
* jacobi_svd: SVD of the small matrix M of step 5 by the
  one-sided (Hestenes) Jacobi method, cyclic-by-rows ordering, no LAPACK.
  Singular values sorted descending; each right singular vector's
  largest-magnitude entry made positive (reading Z10).
"""
from __future__ import annotations

import numpy as np


def householder_qr(Y: np.ndarray):
    """Thin QR, Y (n x l), n >= l.  Returns Q (n x l, orthonormal columns), R (l x l)."""
    A = np.array(Y, dtype=np.float64, copy=True)
    n, l = A.shape
    vs = []
    for j in range(l):
        x = A[j:, j]
        alpha = np.linalg.norm(x)
        v = x.copy()
        if alpha == 0.0:
            vs.append(None)
            continue
        s = 1.0 if x[0] >= 0 else -1.0
        v[0] += s * alpha                      # v = x + sign(x0) ||x|| e1
        v /= np.linalg.norm(v)
        A[j:, j:] -= 2.0 * np.outer(v, v @ A[j:, j:])
        vs.append(v)
    R = np.triu(A[:l, :l])
    Q = np.zeros((n, l))
    Q[:l, :l] = np.eye(l)
    for j in range(l - 1, -1, -1):              # Q = H_0 H_1 ... H_{l-1} [I; 0]
        v = vs[j]
        if v is None:
            continue
        Q[j:, :] -= 2.0 * np.outer(v, v @ Q[j:, :])
    return Q, R


def weighted_gram_schmidt(Y: np.ndarray, Mx):
    """W (n x l) with W^T M W = I and span W = span Y; Mx(X) applies the SPD
    inner-product matrix to the columns of X."""
    Y = np.array(Y, dtype=np.float64, copy=True)
    n, l = Y.shape
    W = np.zeros((n, l))
    for j in range(l):
        v = Y[:, j].copy()
        for _ in range(2):                      # CGS2
            if j > 0:
                r = W[:, :j].T @ Mx(v[:, None])[:, 0]
                v -= W[:, :j] @ r
        nrm = np.sqrt(float(v @ Mx(v[:, None])[:, 0]))
        W[:, j] = v / nrm if nrm > 0 else 0.0
    return W


def jacobi_svd(M: np.ndarray, tol: float = None, max_sweeps: int = 60):
    """One-sided Jacobi: rotate column pairs of A = M until all are mutually
    orthogonal; then M = U diag(s) V^T with U = A/||A_col||, V = accumulated
    rotations.  Returns (U, s, V) with M = U @ diag(s) @ V.T."""
    A = np.array(M, dtype=np.float64, copy=True)
    nr, nc = A.shape
    V = np.eye(nc)
    if tol is None:
        tol = nc * np.finfo(np.float64).eps
    for _ in range(max_sweeps):
        rotated = False
        for p in range(nc - 1):
            for q in range(p + 1, nc):
                ap, aq = A[:, p], A[:, q]
                alpha = ap @ ap
                beta = aq @ aq
                gamma = ap @ aq
                if gamma == 0.0 or abs(gamma) <= tol * np.sqrt(alpha * beta):
                    continue
                rotated = True
                zeta = (beta - alpha) / (2.0 * gamma)
                t = (1.0 if zeta >= 0 else -1.0) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta))
                c = 1.0 / np.sqrt(1.0 + t * t)
                s = c * t
                Ap = A[:, p].copy()
                A[:, p] = c * Ap - s * A[:, q]
                A[:, q] = s * Ap + c * A[:, q]
                Vp = V[:, p].copy()
                V[:, p] = c * Vp - s * V[:, q]
                V[:, q] = s * Vp + c * V[:, q]
        if not rotated:
            break
    else:
        raise RuntimeError("SvdNoConvergence")
    sig = np.sqrt(np.sum(A * A, axis=0))
    order = np.argsort(-sig, kind="stable")
    sig, A, V = sig[order], A[:, order], V[:, order]
    U = np.zeros_like(A)
    nz = sig > 0
    U[:, nz] = A[:, nz] / sig[nz]
    # sign convention (Z10): largest-|.| entry of each right vector positive
    for r in range(nc):
        i = np.argmax(np.abs(V[:, r]))
        if V[i, r] < 0:
            V[:, r] *= -1.0
            U[:, r] *= -1.0
    return U, sig, V
