"""Pins for oracle/parareal.py and oracle/bounds.py against the paper's theorems:
finite termination (proof of Lemma 1), exact coarse solver, the
invariant-subspace identity (Theorem diagonal_convergence), the
Lemma 1 recursion, the a priori and a posteriori
 bounds and the spectral contraction.  The reference
solution is the sequential fine propagation u_{n+1} = F_{n+1} u_n."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import bounds
from oracle.fine import make_op, sequential_reference
from oracle.parareal import parareal
from oracle.rsvd import dense_transfer, delta_eps, exact_truncated, rsvd_interval
from workloads import generators as G
from workloads.configs import C1, get


def _setup(cfg, exact=False):
    op = make_op(cfg)
    if exact:
        F = dense_transfer(op)
        tr = exact_truncated(F, cfg.k)
        truncs = [tr] * cfg.N
    else:
        truncs = [rsvd_interval(op, n, cfg.k, cfg.p, cfg.seed_omega) for n in range(1, cfg.N + 1)]
    if cfg.dim == 1:
        src = G.source_1d(cfg)
        u0 = np.stack([G.initial_value(cfg)] * cfg.nsrc)
        sidx = np.arange(cfg.nsrc)
    else:
        src = G.source_2d(cfg)
        u0 = G.initial_value(cfg)[None]
        sidx = None
    res = parareal(op, truncs, u0, cfg.N, cfg.K, src, sidx)
    ref = sequential_reference(op, u0, cfg.N, src, sidx)
    return op, truncs, res, ref


def _err(res, ref):
    """||e^k_n|| for all k, n (per source): shape (K+1, N+1, nsrc)."""
    d = res.U - ref[None]
    return np.sqrt(np.sum(d.reshape(d.shape[0], d.shape[1], d.shape[2], -1) ** 2, axis=-1))


@pytest.mark.parametrize("name", ["T1", "T4", "T1k1"])
def test_finite_termination(name):
    cfg = get(name)
    _, _, res, ref = _setup(cfg)
    e = _err(res, ref)
    scale = np.max(np.abs(ref))
    for k in range(cfg.K + 1):
        assert np.max(e[k, : k + 1]) <= 1e-13 * scale * np.sqrt(cfg.n_dof)


def test_exact_coarse_solver_converges_immediately():
    """k = n_dof (G = F exactly): u^0 is already the fine solution."""
    cfg = replace(C1, n=20, m=6, k=20, p=0, N=5, K=2)
    _, _, res, ref = _setup(cfg, exact=True)
    e = _err(res, ref)
    assert np.max(e) <= 1e-13 * np.max(np.abs(ref))


def test_invariant_subspace_identity_and_contraction():
    """Time-independent self-adjoint F' with exact truncated-SVD G' (projection
    onto an invariant subspace): e^k_n = (F' - G')^k e^0_{n-k} and
    max_n ||e^k_n|| <= sigma_{R+1}^k max ||e^0_n||."""
    cfg = replace(get("T1"), n=40, k=2, N=8, K=5)
    op, truncs, res, ref = _setup(cfg, exact=True)
    F = dense_transfer(op)
    tr = truncs[0]
    Gp = tr.U @ np.diag(tr.sigma[: cfg.k]) @ tr.V.T
    D = F - Gp
    e = res.U - ref[None]                      # (K+1, N+1, 1, n)
    scale = np.max(np.abs(ref))
    for k in range(cfg.K + 1):
        Dk = np.linalg.matrix_power(D, k)
        for n in range(cfg.N + 1):
            pred = Dk @ e[0, n - k, 0] if n > k else np.zeros(cfg.n)
            assert np.max(np.abs(e[k, n, 0] - pred)) <= 1e-12 * scale
    en = _err(res, ref)[:, :, 0]
    s_next = tr.sigma[cfg.k]
    for k in range(1, cfg.K + 1):
        rhs = bounds.spectral_contraction(s_next, np.max(en[0, 1: cfg.N - k + 1]), k)
        assert np.max(en[k, 1:]) <= rhs * (1 + 1e-10) + 1e-14 * scale


def test_lemma1_and_a_priori_and_a_posteriori_bounds():
    cfg = replace(get("T1"), n=30, k=1, N=8, K=6)
    op, truncs, res, ref = _setup(cfg, exact=True)
    delta, eps = delta_eps(truncs)
    e = _err(res, ref)[:, :, 0]
    floor = 1e-13 * np.max(np.abs(ref))
    bnorm = np.linalg.norm(res.b[:, 0], axis=-1)
    bnorm[0] = np.linalg.norm(res.U[0, 0, 0])          # b_0 := u_0
    for k in range(0, cfg.K + 1):
        for n in range(1, cfg.N + 1):
            if k >= 1:
                # Lemma 1
                assert e[k, n] <= eps * e[k - 1, n - 1] + delta * e[k, n - 1] + floor
                # eq. error_bound_eps_delta and the a posteriori bound
                assert e[k, n] <= bounds.a_priori_from_e0(delta, eps, e[0], n, k) + floor
                assert e[k, n] <= bounds.a_posteriori(delta, eps, res.upd[k, :, 0], n) + floor
            # eq. error_bound_initial / eps_delta2
            assert e[k, n] <= bounds.a_priori_k(delta, eps, bnorm, n, k) + floor
        if k >= 1:
            assert np.max(e[k, 1:]) <= bounds.a_posteriori_sup(delta, eps, res.upd[k, :, 0]) + floor
            # eqs. error_bound_eps (delta <= 1) and error_bound_eps_inf_time (delta < 1)
            assert delta < 1
            assert np.max(e[k, 1:]) <= bounds.a_priori_eps(eps, cfg.N, k, e[0]) + floor
            assert np.max(e[k, 1:]) <= bounds.a_priori_eps_inf_time(delta, eps, cfg.N, k, e[0]) + floor


def test_update_norms_are_iterate_differences():
    cfg = get("T4")
    _, _, res, _ = _setup(cfg)
    d = res.U[1:] - res.U[:-1]
    ref = np.sqrt(np.sum(d ** 2, axis=-1))
    np.testing.assert_allclose(res.upd[1:], ref, rtol=1e-14, atol=0)
    assert np.all(res.upd[1:, 0] == 0)                 # u^k_0 = u_0 always


def test_parareal_converges_2d_small():
    cfg = replace(get("T2D"), n=15, N=5, K=5)
    _, _, res, ref = _setup(cfg)
    e = _err(res, ref)[:, :, 0]
    assert np.max(e[cfg.K]) <= 1e-12 * np.max(np.abs(ref))
    assert np.max(e[0]) > 1e-8 * np.max(np.abs(ref))   # the iteration had work to do
