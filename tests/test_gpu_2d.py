"""GPU parity of the 2D separable path (K2, FP64 tensor cores) against the
oracle (x-sine transform + Thomas lines, itself pinned to dense solves).
Tolerance 1e-8 normwise on the 2D GEMM paths (BASELINE.json north_star)."""
from dataclasses import replace

import numpy as np
import pytest

from gpu_util import TAU_2D, empty_batch, from_gpu, gpu_op, gpu_source, relnorm, to_gpu
from oracle.fine import fine, make_op, sequential_reference
from oracle.parareal import parareal as oracle_parareal
from oracle.rng import gaussian_sketch
from oracle.rsvd import rsvd_interval
from workloads import generators as G
from workloads.configs import C3, get

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    from paper_2508_08873_b200 import build as B
    B.build()
    assert torch.cuda.is_available()


def test_sketch_2d_interior_numbering():
    cfg = get("T2D")
    op = gpu_op(cfg)
    l, nint, q0 = 5, 2, 3
    out = empty_batch(cfg, nint * l)
    op.gaussian_sketch(q0, nint, l, 77, out)
    got = from_gpu(cfg, out)                                # (nvec, n, n) interior
    for j in range(nint):
        ref = gaussian_sketch(77, q0 + j, cfg.n * cfg.n, l)  # row = ix*n + iy
        for c in range(l):
            np.testing.assert_allclose(got[j * l + c].ravel(), ref[:, c], rtol=0, atol=1e-14)
    ghost = out.view(nint * l, cfg.n + 1, cfg.n + 1)
    assert float(ghost[:, 0, :].abs().max()) == 0.0 and float(ghost[:, :, 0].abs().max()) == 0.0


@pytest.mark.parametrize("name,n,m,B", [("T2D", 63, 10, 5), ("T2D", 127, 3, 3), ("C3", 255, 128, 3)])
@pytest.mark.parametrize("mode", ["linear", "adjoint"])
def test_fine_2d_linear(name, n, m, B, mode):
    from paper_2508_08873_b200 import PR_ADJOINT, PR_LINEAR
    cfg = replace(get(name), n=n, m=m)
    op_o, op_g = make_op(cfg), gpu_op(cfg)
    X = np.random.default_rng(n + m).standard_normal((B, n, n))
    out = empty_batch(cfg, B)
    op_g.fine_propagate(PR_LINEAR if mode == "linear" else PR_ADJOINT, 1, m, to_gpu(cfg, X), out)
    got = from_gpu(cfg, out)
    ref = fine(op_o, 2, X, mode)
    for v in range(B):
        assert relnorm(got[v], ref[v]) <= TAU_2D * 1e-3, v       # expect ~1e-14
    P = n + 1
    o = out.view(B, P, P)
    assert float(o[:, 0, :].abs().max()) == 0.0 and float(o[:, :, 0].abs().max()) == 0.0


@pytest.mark.parametrize("name,nb", [("T2D", 1), ("T2D", 4), ("C3", 1)])
def test_fine_2d_affine_and_offset(name, nb):
    from paper_2508_08873_b200 import PR_AFFINE, PR_LINEAR
    cfg = replace(get(name), source="bump4" if nb == 4 else "bump1")
    if name == "C3":
        cfg = replace(cfg, N=4)
    op_o, op_g = make_op(cfg), gpu_op(cfg)
    src_g = gpu_source(cfg)
    src_o = G.source_2d(cfg)
    B = 3
    X = np.random.default_rng(1).standard_normal((B, cfg.n, cfg.n))
    q0 = 1
    # b_q = F_q 0 (zero input), one vector per interval
    bq = empty_batch(cfg, B)
    op_g.fine_propagate(PR_AFFINE, q0, cfg.m, None, bq, vecs_per_interval=1, source=src_g)
    gotb = from_gpu(cfg, bq)
    for v in range(B):
        ref = fine(op_o, q0 + v + 1, np.zeros((cfg.n, cfg.n)), "affine", src_o)
        assert relnorm(gotb[v], ref) <= TAU_2D * 1e-3
    # F_q x = F_q' x + b_q, through PR_AFFINE with input and through the offset path
    out = empty_batch(cfg, B)
    op_g.fine_propagate(PR_AFFINE, q0, cfg.m, to_gpu(cfg, X), out, vecs_per_interval=1, source=src_g)
    out2 = empty_batch(cfg, B)
    op_g.fine_propagate(PR_LINEAR, q0, cfg.m, to_gpu(cfg, X), out2, offset=bq)
    g1, g2 = from_gpu(cfg, out), from_gpu(cfg, out2)
    for v in range(B):
        ref = fine(op_o, q0 + v + 1, X[v], "affine", src_o)
        assert relnorm(g1[v], ref) <= TAU_2D * 1e-3
        assert relnorm(g2[v], ref) <= TAU_2D * 1e-3


def _check_interval_2d(cfg, Gg, q, info, probes=4):
    op_o = make_op(cfg)
    tr = rsvd_interval(op_o, q + 1, cfg.k, cfg.p, cfg.seed_omega)
    s1 = tr.sigma[0]
    assert np.max(np.abs(info["sigma"][q] - tr.sigma)) <= TAU_2D * s1
    X = np.random.default_rng(q).standard_normal((probes, cfg.n, cfg.n))
    Y = empty_batch(cfg, probes)
    Gg.apply(q, to_gpu(cfg, X), Y, 2)
    got = from_gpu(cfg, Y).reshape(probes, -1)
    ref = tr.apply_linear(X.reshape(probes, -1))
    for v in range(probes):
        assert np.linalg.norm(got[v] - ref[v]) <= TAU_2D * s1 * np.linalg.norm(X[v])


def test_build_2d_small_all_intervals():
    from paper_2508_08873_b200 import Coarse
    cfg = get("T2D")
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    for q in range(cfg.N):
        _check_interval_2d(cfg, Gg, q, info)


def test_build_c3_sampled_intervals():
    from paper_2508_08873_b200 import Coarse
    cfg = C3
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    for q in (0, cfg.N - 1):
        _check_interval_2d(cfg, Gg, q, info)


def _parareal_2d(cfg, hist_on=True):
    import torch
    from paper_2508_08873_b200 import Coarse, parareal
    opg = gpu_op(cfg)
    Gg = Coarse.build(opg, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    u0 = G.initial_value(cfg)[None]
    Uo = empty_batch(cfg, cfg.N + 1)
    hist = torch.zeros((cfg.K + 1,) + tuple(Uo.shape), dtype=torch.float64, device="cuda") if hist_on else None
    upd, bn = parareal(Gg, opg, to_gpu(cfg, u0), gpu_source(cfg), cfg.K, Uo, nsrc=1, hist=hist)
    _parareal_2d.last_info = Gg.info()
    return Uo, hist, upd, bn, u0


def test_parareal_2d_small_all_iterates():
    cfg = get("T2D")
    Uo, hist, upd, bn, u0 = _parareal_2d(cfg)
    op_o = make_op(cfg)
    truncs = [rsvd_interval(op_o, n, cfg.k, cfg.p, cfg.seed_omega) for n in range(1, cfg.N + 1)]
    res = oracle_parareal(op_o, truncs, u0, cfg.N, cfg.K, G.source_2d(cfg))
    scale = np.max(np.abs(res.U))
    for k in range(cfg.K + 1):
        got = from_gpu(cfg, hist[k])
        err = np.max(np.abs(got - res.U[k][:, 0]))
        assert err <= TAU_2D * scale, (k, err / scale)
    assert np.max(np.abs(upd[:, :, 0] - res.upd[1:, :, 0])) <= TAU_2D * scale
    # the iteration converges to the fine solution
    ref = sequential_reference(op_o, u0, cfg.N, G.source_2d(cfg))
    assert np.max(np.abs(from_gpu(cfg, Uo) - ref[:, 0])) <= 1e-9 * scale


def test_parareal_c3_against_fine_solution():
    cfg = C3
    Uo, hist, upd, bn, u0 = _parareal_2d(cfg, hist_on=False)
    op_o = make_op(cfg)
    ref = sequential_reference(op_o, u0, cfg.N, G.source_2d(cfg))[:, 0]
    got = from_gpu(cfg, Uo)
    scale = np.max(np.linalg.norm(ref.reshape(cfg.N + 1, -1), axis=1))
    err = np.linalg.norm((got - ref).reshape(cfg.N + 1, -1), axis=1)
    # finite termination: u^K_n = u_n for n <= K
    assert np.max(err[: cfg.K + 1]) <= TAU_2D * scale
    # beyond: the Parareal error after K = 8 iterations (~1e-13 relative at k >= 4)
    assert np.max(err) <= 1e-9 * scale


def test_build_c5_shard_sampled_intervals():
    """C5 (511^2 grid, N = 512) does not fit one GPU (205 GB of factors).  One
    B200 builds the shard of intervals one of eight ranks owns; intervals are
    independent and seeded by (seed, q, column), so the shard must agree with
    the oracle's rSVD of the same intervals."""
    from paper_2508_08873_b200 import Coarse
    from workloads.configs import C5
    cfg = C5
    first, nloc = 448, 8                       # a slice of rank 7's intervals
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega,
                      first_interval=first, n_local=nloc)
    info = Gg.info()
    op_o = make_op(cfg)
    for ql in (0, nloc - 1):
        tr = rsvd_interval(op_o, first + ql + 1, cfg.k, cfg.p, cfg.seed_omega)
        s1 = tr.sigma[0]
        assert np.max(np.abs(info["sigma"][ql] - tr.sigma)) <= TAU_2D * s1
        X = np.random.default_rng(ql).standard_normal((2, cfg.n, cfg.n))
        Y = empty_batch(cfg, 2)
        Gg.apply(ql, to_gpu(cfg, X), Y, 2)
        got = from_gpu(cfg, Y).reshape(2, -1)
        ref = tr.apply_linear(X.reshape(2, -1))
        for v in range(2):
            assert np.linalg.norm(got[v] - ref[v]) <= TAU_2D * s1 * np.linalg.norm(X[v])


def test_lifted_factors_orthonormal_2d():
    import torch
    from paper_2508_08873_b200 import Coarse
    cfg = C3
    op = gpu_op(cfg)
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    U = torch.empty((op.rows, cfg.k), dtype=torch.float64, device="cuda")
    V = torch.empty_like(U)
    I = torch.eye(cfg.k, dtype=torch.float64, device="cuda")
    for q in (0, cfg.N - 1):
        Gc.export_interval(q, U_q=U, V_q=V)
        assert float((U.T @ U - I).abs().max()) < 1e-13
        assert float((V.T @ V - I).abs().max()) < 1e-13
        P = cfg.n + 1
        assert float(U.view(P, P, cfg.k)[0].abs().max()) == 0.0      # ghosts stay zero


def _parareal_vs_oracle_iterates(cfg, kmax, tau):
    """Every iterate u^k_n, k <= kmax, and the update norms of the GPU's
    Parareal (reduced sweep) against the oracle's direct form on
    the oracle's own per-interval rSVDs (parallel worker pool)."""
    from oracle_pool import rsvd_intervals
    Uo, hist, upd, bn, u0 = _parareal_2d(cfg)
    info = _parareal_2d.last_info
    truncs = rsvd_intervals(cfg)
    sig = np.stack([t.sigma for t in truncs])
    assert np.max(np.abs(info["sigma"] - sig)) <= tau * sig.max()
    op_o = make_op(cfg)
    res = oracle_parareal(op_o, truncs, u0, cfg.N, kmax, G.source_2d(cfg))
    scale = np.max(np.linalg.norm(res.U.reshape(kmax + 1, cfg.N + 1, -1), axis=-1))
    errs = []
    for k in range(kmax + 1):
        got = from_gpu(cfg, hist[k]).reshape(cfg.N + 1, -1)
        err = np.max(np.linalg.norm(got - res.U[k][:, 0].reshape(cfg.N + 1, -1), axis=-1))
        errs.append(err / scale)
        assert err <= tau * scale, (k, err / scale)
    assert np.max(np.abs(upd[:kmax, :, 0] - res.upd[1:kmax + 1, :, 0])) <= tau * scale
    return errs, res


@pytest.mark.timeout(1200)
def test_parareal_c3_iterates_k0_to_3_match_oracle():
    """C3 is the configuration whose Parareal really iterates (SURVEY A.5:
    relative error 4e-4 at k = 0 to ~1e-10 at k = 2): iterates 0..3 of the
    full-size run against the oracle's direct form."""
    from dataclasses import replace as _r
    cfg = _r(C3, K=3)
    errs, res = _parareal_vs_oracle_iterates(cfg, 3, TAU_2D)
    # the iteration really moves: the k = 0 iterate is far from the converged one
    scale = np.max(np.abs(res.U))
    assert np.max(np.abs(res.U[0] - res.U[3])) > 1e-6 * scale


@pytest.mark.timeout(1800)
def test_parareal_c5_geometry_matches_oracle():
    """C5's 511^2 grid, k = 96, p = 16 on 16 intervals: build and all Parareal
    iterates against the oracle (BASELINE.json configs[4] geometry)."""
    from workloads.configs import get as _get
    cfg = _get("C5G")
    _parareal_vs_oracle_iterates(cfg, cfg.K, TAU_2D)


@pytest.mark.parametrize("q,indep", [(1, False), (0, True)])
def test_build_2d_rsvd_variants_match_oracle(q, indep):
    from paper_2508_08873_b200 import Coarse
    cfg = get("T2D")
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega, power_iterations=q,
                      independent_adjoint=indep)
    info = Gg.info()
    op_o = make_op(cfg)
    for qi in (0, cfg.N - 1):
        tr = rsvd_interval(op_o, qi + 1, cfg.k, cfg.p, cfg.seed_omega, power_iterations=q,
                           independent_adjoint=indep)
        s1 = tr.sigma[0]
        assert np.max(np.abs(info["sigma"][qi] - tr.sigma)) <= TAU_2D * s1
        X = np.random.default_rng(qi).standard_normal((2, cfg.n, cfg.n))
        Y = empty_batch(cfg, 2)
        Gg.apply(qi, to_gpu(cfg, X), Y, 2)
        got = from_gpu(cfg, Y).reshape(2, -1)
        ref = tr.apply_linear(X.reshape(2, -1))
        for v in range(2):
            assert np.linalg.norm(got[v] - ref[v]) <= TAU_2D * s1 * np.linalg.norm(X[v])


@pytest.mark.timeout(1800)
def test_c5_power_iteration_build_matches_oracle():
    """C5's slowly decaying spectrum is where q >= 1 matters:
    the GPU build with q = 1 on two C5-geometry intervals against the oracle."""
    from paper_2508_08873_b200 import Coarse
    from workloads.configs import get as _get
    cfg = _get("C5G")
    first, nloc = 6, 2
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega, first_interval=first,
                      n_local=nloc, power_iterations=1)
    info = Gg.info()
    op_o = make_op(cfg)
    for ql in range(nloc):
        tr = rsvd_interval(op_o, first + ql + 1, cfg.k, cfg.p, cfg.seed_omega, power_iterations=1)
        assert np.max(np.abs(info["sigma"][ql] - tr.sigma)) <= TAU_2D * tr.sigma[0]
