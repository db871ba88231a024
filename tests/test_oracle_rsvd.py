"""Pins for oracle/rsvd.py against closed-form spectra, dense SVDs
and the truncation identity ||F' - G'|| = sigma_{R+1} (eq. truncation_error)."""
from dataclasses import replace

import numpy as np

from oracle.fine import Op1D, make_op
from oracle.linalg import householder_qr, jacobi_svd
from oracle.rng import gaussian_sketch
from oracle.rsvd import dense_transfer, rsvd_interval
from workloads.configs import C1, C2, C3, get


def _closed_form_1d(cfg):
    j = np.arange(1, cfg.n + 1)
    lam = 4.0 / cfg.h ** 2 * np.sin(j * np.pi * cfg.h / 2) ** 2
    return np.sort((1 + cfg.dt * lam) ** (-cfg.m))[::-1]


def test_c1_sigma_closed_form_and_truncation_identity():
    cfg = C1
    op = make_op(cfg)
    tr = rsvd_interval(op, 3, cfg.k, cfg.p, cfg.seed_omega)
    ref = _closed_form_1d(cfg)
    assert np.max(np.abs(tr.sigma[: cfg.k] - ref[: cfg.k])) <= 1e-14 * ref[0]
    F = dense_transfer(op)
    Gd = tr.U @ np.diag(tr.sigma[: cfg.k]) @ tr.V.T
    err = np.linalg.norm(F - Gd, 2)
    # eq. truncation_error: ||F - G|| = sigma_{R+1} (here at the rounding floor)
    assert err <= ref[cfg.k] + 1e-14 * ref[0]
    # interlacing: computed sigma never exceeds the exact ones
    assert np.all(tr.sigma <= ref[: cfg.l] + 1e-13 * ref[0])


def test_rsvd_exact_for_full_sketch_tiny_grid():
    """k = n, p = 0: W = V = R^n so G' = F' exactly and all sigma are exact."""
    cfg = replace(C1, n=15, m=3, k=15, p=0)
    op = make_op(cfg)
    tr = rsvd_interval(op, 1, cfg.k, cfg.p, 7)
    F = dense_transfer(op)
    np.testing.assert_allclose(tr.sigma, np.linalg.svd(F, compute_uv=False), rtol=0, atol=1e-14)
    np.testing.assert_allclose(tr.U @ np.diag(tr.sigma) @ tr.V.T, F, rtol=0, atol=1e-14)


def test_rsvd_nonsymmetric_truncation_identity_and_swapped_reading():
    """Non-normal F' (like Exp 2).  With the swapped psi/phi reading
    (Z5) ||F' - G'|| matches sigma_{k+1} of F'; the literal P:293-294
    assignment does not give the SVD of P_W F'."""
    rng = np.random.default_rng(11)
    n = 60
    sub = -30.0 - 20 * rng.uniform(0, 1, n)
    sup = -10.0 - 5 * rng.uniform(0, 1, n)
    diag = -(sub + sup) + 1.0 + rng.uniform(0, 1, n)
    sub[0] = 0
    sup[-1] = 0
    op = Op1D(sub, diag, sup, dt=0.2, m=10)
    k, p = 5, 10
    tr = rsvd_interval(op, 1, k, p, 99)
    F = dense_transfer(op)
    s = np.linalg.svd(F, compute_uv=False)
    err = np.linalg.norm(F - tr.U @ np.diag(tr.sigma[:k]) @ tr.V.T, 2)
    assert abs(err - s[k]) <= 1e-12 * s[0]
    assert np.max(np.abs(tr.sigma[:k] - s[:k])) <= 1e-8 * s[0]
    # literal reading: psi from V-basis, phi from W-basis
    l = k + p
    Om = gaussian_sketch(99, 0, n, l)
    W, _ = householder_qr(F @ Om)
    Z = F.T @ W
    Vb, _ = householder_qr(Z)
    Psi, sg, Phi = jacobi_svd(Z.T @ Vb)
    lit = (Vb @ Psi[:, :k]) @ np.diag(sg[:k]) @ (W @ Phi[:, :k]).T
    assert np.linalg.norm(F - lit, 2) > 10 * s[k]


def test_c2_sigma_closed_form():
    cfg = replace(C2, N=64)
    op = make_op(cfg)
    tr = rsvd_interval(op, 64, cfg.k, cfg.p, cfg.seed_omega)
    ref = _closed_form_1d(cfg)
    # m = 256 steps, each with O(u) relative rounding: m * u ~ 6e-14 (reading R-ACC)
    assert np.max(np.abs(tr.sigma[: cfg.k] - ref[: cfg.k])) <= 2e-13 * ref[0]
    assert abs(tr.sigma[0] - 0.8571) < 1e-4


def test_2d_rsvd_tiny_grid_against_dense():
    """l = n_dof: the sketch spans V, so all sigma and G' are exact."""
    cfg = replace(C3, n=7, m=6, k=30, p=19)
    op = make_op(cfg)
    tr = rsvd_interval(op, 2, cfg.k, cfg.p, 5)
    F = dense_transfer(op)
    s = np.linalg.svd(F, compute_uv=False)
    np.testing.assert_allclose(tr.sigma, s, rtol=0, atol=1e-14 * s[0])
    err = np.linalg.norm(F - tr.U @ np.diag(tr.sigma[: cfg.k]) @ tr.V.T, 2)
    assert abs(err - s[cfg.k]) <= 1e-13 * s[0]


def test_2d_rsvd_interlacing_and_top_sigma():
    """Randomized sigma never exceed the exact ones (projection); with fast
    decay (long interval) the leading ones are accurate."""
    cfg = replace(C3, n=11, m=40, T=8.0, N=8, k=10, p=10)
    op = make_op(cfg)
    tr = rsvd_interval(op, 1, cfg.k, cfg.p, 3)
    s = np.linalg.svd(dense_transfer(op), compute_uv=False)
    assert np.all(tr.sigma <= s[: cfg.l] + 1e-13 * s[0])
    assert np.max(np.abs(tr.sigma[:4] - s[:4])) <= 1e-8 * s[0]


def test_fine_spectrum_converges_to_paper_fourier_formula():
    """the exact transfer operator of the 1D Dirichlet heat equation has
    sigma_j = exp(-j^2 pi^2 dT).  The oracle's backward-Euler F' must approach it
    at first order in dt (golden: tests/golden/paper_exp1_fourier_sigma.txt)."""
    import os
    rows = np.loadtxt(os.path.join(os.path.dirname(__file__), "golden",
                                   "paper_exp1_fourier_sigma.txt"))
    errs = []
    for m in (64, 128, 256):
        cfg = replace(C1, n=127, m=m)
        s = np.linalg.svd(dense_transfer(make_op(cfg)), compute_uv=False)
        errs.append(np.abs(s[:3] - rows[:3, 2]))
    errs = np.array(errs)
    assert np.all(errs[-1] < 0.08 * rows[:3, 2])
    ratio = errs[:-1] / errs[1:]
    assert np.all(ratio > 1.7) and np.all(ratio < 2.2)
