"""Pins of the oracle's reporting functions: the
estimator efficiency eq. def_efficiency (hand-evaluated), the max-over-time
error against brute-force dense partial products and its
invariants, and classical Parareal with G = 0 / exact G / a coarse Euler
step against closed forms and finite termination
(P:391-392)."""
import numpy as np
import pytest

from oracle.bounds import efficiency
from oracle.fine import dense_step_product, fine, fine_trajectory, make_op, sequential_reference
from oracle.parareal import parareal as parareal_spectral
from oracle.parareal import parareal_classical, trajectory_error
from oracle.rsvd import rsvd_interval
from workloads import generators as G
from workloads.configs import get


def test_efficiency_hand_evaluated():
    """N = 4, delta = 1/2, eps = 1/10, ||u^k_m - u^{k-1}_m|| = (0, 1, 2, 4, 8):
    denominators (n = 1, 2, 3) = 0, 0.1 * 1, 0.1 * (0.5 * 1 + 2) = 0.25 -> max 0.25
    (n = N = 4 excluded as printed); eta = 0.05 / 0.25 = 0.2."""
    upd = np.array([0.0, 1.0, 2.0, 4.0, 8.0])
    assert abs(efficiency(0.5, 0.1, upd, 0.05, 4) - 0.2) < 1e-15


@pytest.mark.parametrize("name", ["E2", "T1"])
def test_trajectory_error_invariants(name):
    cfg = get(name)
    op = make_op(cfg)
    src = G.source_1d(cfg)
    u0 = np.asarray(G.initial_value(cfg))[None, :]
    ref = sequential_reference(op, u0, cfg.N, src)
    assert np.all(trajectory_error(op, ref, ref, cfg.N, src) == 0.0)
    rng = np.random.default_rng(2)
    Uk = ref + 1e-3 * rng.standard_normal(ref.shape)
    Uk[0] = ref[0]
    te = trajectory_error(op, Uk, ref, cfg.N, src)[0]
    bnd = max(np.linalg.norm(Uk[n] - ref[n]) for n in range(cfg.N))
    end = np.linalg.norm(fine(op, cfg.N, Uk[cfg.N - 1], "affine", src) - ref[cfg.N])
    assert te >= bnd * (1 - 1e-12) and te >= end * (1 - 1e-12)


def test_trajectory_error_matches_dense_partial_products():
    """The error inside interval n is F'_{n,j} e_{n-1} with the dense partial
    products of the step matrices (E2, brute force)."""
    cfg = get("E2")
    op = make_op(cfg)
    src = G.source_1d(cfg)
    u0 = np.asarray(G.initial_value(cfg))[None, :]
    ref = sequential_reference(op, u0, cfg.N, src)
    rng = np.random.default_rng(5)
    Uk = ref + rng.standard_normal(ref.shape)
    Uk[0] = ref[0]
    best = 0.0
    for n in range(1, cfg.N + 1):
        e = (Uk[n - 1] - ref[n - 1])[0]
        for j in range(0, cfg.m + (1 if n == cfg.N else 0)):
            if j == 0:
                v = e
            else:
                # partial product of steps g0+1..g0+j: an interval of length j starting at g0
                g0 = (n - 1) * cfg.m
                P = np.eye(cfg.n)
                Md = np.diag(op.M[1]) + np.diag(op.M[0][1:], -1) + np.diag(op.M[2][:-1], 1)
                for g in range(g0 + 1, g0 + j + 1):
                    a, d, c = (arr[g - 1] for arr in op.L)
                    Lg = np.diag(d) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
                    P = np.linalg.solve(Lg, Md @ P)
                v = P @ e
            best = max(best, np.linalg.norm(v))
    te = trajectory_error(op, Uk, ref, cfg.N, src)[0]
    assert abs(te - best) <= 1e-12 * best


def test_fine_trajectory_ends_at_fine():
    cfg = get("E2FD")
    op = make_op(cfg)
    src = G.source_1d(cfg)
    x = np.random.default_rng(1).standard_normal((2, cfg.n))
    tr = fine_trajectory(op, 4, x, src)
    assert len(tr) == cfg.m + 1
    assert np.linalg.norm(tr[-1] - fine(op, 4, x, "affine", src)) <= 1e-14 * np.linalg.norm(tr[-1])


@pytest.mark.parametrize("name", ["E2", "T1"])
def test_classical_parareal_zero_coarse(name):
    """G = 0: u^0_n = 0 (n >= 1), u^1_1 = F_1 u0, u^1_n = F_n 0 = b_n (n >= 2),
    and finite termination u^k_n = u_n for n <= k."""
    cfg = get(name)
    op = make_op(cfg)
    src = G.source_1d(cfg)
    u0 = np.asarray(G.initial_value(cfg))[None, :]
    res = parareal_classical(op, lambda n, x: np.zeros_like(x), u0, cfg.N, 4, src)
    assert np.all(res.U[0, 1:] == 0.0)
    ref = sequential_reference(op, u0, cfg.N, src)
    assert np.linalg.norm(res.U[1, 1] - ref[1]) <= 1e-14 * np.linalg.norm(ref[1])
    for n in range(2, cfg.N + 1):
        b = fine(op, n, np.zeros_like(u0), "affine", src)
        assert np.linalg.norm(res.U[1, n] - b) <= 1e-13 * max(np.linalg.norm(b), 1e-300)
    for k in range(5):
        for n in range(k + 1):
            assert np.linalg.norm(res.U[k, n] - ref[n]) <= 1e-12 * np.linalg.norm(ref[n]) + 1e-300


def test_classical_parareal_exact_coarse_and_spectral_agree():
    """G = F (the exact propagator): u^0 is the sequential solution; and the
    classical routine with G_n = G_n' + b_n reproduces the spectral oracle."""
    cfg = get("T1")
    op = make_op(cfg)
    src = G.source_1d(cfg)
    u0 = np.asarray(G.initial_value(cfg))[None, :]
    ref = sequential_reference(op, u0, cfg.N, src)
    ex = parareal_classical(op, lambda n, x: fine(op, n, x, "affine", src), u0, cfg.N, 2, src)
    assert np.max(np.abs(ex.U[0] - ref)) <= 1e-13 * np.max(np.abs(ref))
    truncs = [rsvd_interval(op, n, cfg.k, cfg.p, cfg.seed_omega) for n in range(1, cfg.N + 1)]
    sp = parareal_spectral(op, truncs, u0, cfg.N, 3, src)
    Gf = lambda n, x: truncs[n - 1].apply_linear(x) + sp.b[n]
    cl = parareal_classical(op, Gf, u0, cfg.N, 3, src)
    assert np.max(np.abs(cl.U - sp.U)) <= 1e-12 * np.max(np.abs(sp.U))
