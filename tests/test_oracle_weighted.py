"""Pins of the oracle's rSVD in the mass-matrix inner product (SURVEY 8(f)
row 2; the generalized SVD of eq. svd) to independent library
computations: the singular values of C F' C^{-1} (scipy Cholesky + numpy SVD),
exactness for l = n, M-orthonormal singular vectors, and the truncation
error ||F' - G'||_M = sigma_{R+1} (eq. truncation_error)."""
import numpy as np
import scipy.linalg

from oracle.fine import dense_step_product, make_op
from oracle.rsvd import rsvd_interval
from workloads.configs import get


def _mass(op):
    ms, md, mp = op.M
    return np.diag(md) + np.diag(ms[1:], -1) + np.diag(mp[:-1], 1)


def test_weighted_rsvd_is_the_generalized_svd():
    # a coarse Exp 2 grid (11 nodes, 2 steps per interval): no singular value
    # underflows, so l = n is a well-posed exact SVD
    from dataclasses import replace
    cfg = replace(get("E2"), n=11, m=2)
    op = make_op(cfg)
    M = _mass(op)
    C = scipy.linalg.cholesky(M)                  # upper, M = C^T C
    F = dense_step_product(op, 3)
    ref = np.linalg.svd(C @ F @ np.linalg.inv(C), compute_uv=False)
    t = rsvd_interval(op, 3, cfg.n, 0, cfg.seed_omega, inner=op.M)      # l = n: exact
    assert np.max(np.abs(t.sigma - ref)) <= 1e-12 * ref[0]
    # psi M-orthonormal, G' = F' (full rank), and the k-truncation error in the M norm
    assert np.max(np.abs(t.U.T @ M @ t.U - np.eye(cfg.n))) < 1e-10
    Gfull = t.U @ np.diag(t.sigma) @ t.V.T
    assert np.linalg.norm(Gfull - F, 2) <= 1e-11 * np.linalg.norm(F, 2)
    k = 4
    assert ref[k] > 1e-6
    Gk = t.U[:, :k] @ np.diag(t.sigma[:k]) @ t.V[:, :k].T
    errM = np.linalg.norm(C @ (F - Gk) @ np.linalg.inv(C), 2)
    assert abs(errM - ref[k]) <= 1e-10 * ref[0]


def test_weighted_rsvd_small_rank_top_values():
    """rank-5 sketch with p = 1 (the paper's Exp 2 choice): the leading
    generalized singular values to the sketch accuracy, sigma_1 = 1 (the
    undamped constant mode is M-normalisable: F' 1 = 1)."""
    cfg = get("E2")
    op = make_op(cfg)
    C = scipy.linalg.cholesky(_mass(op))
    F = dense_step_product(op, 5)
    ref = np.linalg.svd(C @ F @ np.linalg.inv(C), compute_uv=False)
    t = rsvd_interval(op, 5, cfg.k, cfg.p, cfg.seed_omega, inner=op.M)
    assert abs(t.sigma[0] - ref[0]) <= 1e-10 * ref[0]
    assert abs(ref[0] - 1.0) < 1e-12
