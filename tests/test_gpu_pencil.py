"""GPU parity of the time-dependent pencil path (the
paper's Experiment 2) against the oracle, through the C ABI:
fine propagation (LINEAR / ADJOINT in reverse step order / AFFINE), the rSVD
build of every interval, and the Parareal iterates.  Tolerance: BASELINE.json
north_star, 1e-10 normwise (reading Z11)."""
import numpy as np
import pytest

from gpu_util import TAU_1D, empty_batch, from_gpu, gpu_op, gpu_source, to_gpu
from oracle.fine import fine, make_op
from oracle.parareal import parareal as oracle_parareal
from oracle.rsvd import rsvd_interval
from workloads import generators as G
from workloads.configs import get

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    from paper_2508_08873_b200 import build as B
    B.build()
    assert torch.cuda.is_available()


@pytest.mark.parametrize("name", ["E2", "E2FD", "E2L"])
@pytest.mark.parametrize("mode", ["linear", "adjoint", "affine"])
def test_pencil_fine_matches_oracle(name, mode):
    from paper_2508_08873_b200 import PR_ADJOINT, PR_AFFINE, PR_LINEAR
    cfg = get(name)
    op = gpu_op(cfg)
    op_o = make_op(cfg)
    rng = np.random.default_rng(11)
    vpi = 3
    q0 = cfg.N - 4 if cfg.N > 4 else 0
    nint = 3
    X = rng.standard_normal((nint * vpi, cfg.n))
    Y = empty_batch(cfg, nint * vpi)
    src = gpu_source(cfg) if mode == "affine" else None
    m = {"linear": PR_LINEAR, "adjoint": PR_ADJOINT, "affine": PR_AFFINE}[mode]
    op.fine_propagate(m, q0, cfg.m, to_gpu(cfg, X), Y, vecs_per_interval=vpi, source=src)
    got = from_gpu(cfg, Y)
    for j in range(nint):
        ref = fine(op_o, q0 + j + 1, X[j * vpi:(j + 1) * vpi], mode,
                   G.source_1d(cfg) if mode == "affine" else None)
        sl = got[j * vpi:(j + 1) * vpi]
        for v in range(vpi):
            assert np.linalg.norm(sl[v] - ref[v]) <= TAU_1D * np.linalg.norm(ref[v]), (j, v)


def test_pencil_intervals_beyond_steps_rejected():
    from paper_2508_08873_b200 import PR_LINEAR
    from paper_2508_08873_b200._lib import PrError
    cfg = get("E2")
    op = gpu_op(cfg)
    Y = empty_batch(cfg, 2)
    with pytest.raises(PrError):
        op.fine_propagate(PR_LINEAR, cfg.N, cfg.m, None, Y, vecs_per_interval=1)


@pytest.mark.parametrize("name", ["E2", "E2FD"])
def test_pencil_build_matches_oracle(name):
    from paper_2508_08873_b200 import Coarse
    cfg = get(name)
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    op_o = make_op(cfg)
    for q in range(cfg.N):
        tr = rsvd_interval(op_o, q + 1, cfg.k, cfg.p, cfg.seed_omega)
        s1 = tr.sigma[0]
        assert s1 >= 1.0 - 1e-12                    # undamped constant mode (Neumann)
        assert np.max(np.abs(info["sigma"][q] - tr.sigma)) <= TAU_1D * s1, q
        X = np.random.default_rng(q).standard_normal((4, cfg.n))
        Y = empty_batch(cfg, 4)
        Gg.apply(q, to_gpu(cfg, X), Y, 1)
        got, ref = from_gpu(cfg, Y), tr.apply_linear(X)
        for v in range(4):
            assert np.linalg.norm(got[v] - ref[v]) <= TAU_1D * s1 * np.linalg.norm(X[v]), (q, v)


def test_pencil_build_large_sampled_intervals():
    """E2L (4096 nodes, 64 x 64 steps): sampled intervals of a full build."""
    from paper_2508_08873_b200 import Coarse
    cfg = get("E2L")
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    op_o = make_op(cfg)
    for q in (0, 31, 63):
        tr = rsvd_interval(op_o, q + 1, cfg.k, cfg.p, cfg.seed_omega)
        assert np.max(np.abs(info["sigma"][q] - tr.sigma)) <= TAU_1D * tr.sigma[0], q


@pytest.mark.parametrize("name", ["E2", "E2FD"])
def test_pencil_parareal_iterates_match_oracle(name):
    import torch
    from paper_2508_08873_b200 import Coarse, parareal
    cfg = get(name)
    op = gpu_op(cfg)
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    u0 = G.initial_value(cfg)[None, :]
    op_o = make_op(cfg)
    truncs = [rsvd_interval(op_o, q, cfg.k, cfg.p, cfg.seed_omega) for q in range(1, cfg.N + 1)]
    for K in (0, 1, 3):
        Uo = torch.zeros((cfg.n, cfg.N + 1), dtype=torch.float64, device="cuda")
        u0g = torch.tensor(np.ascontiguousarray(u0.T), dtype=torch.float64, device="cuda")
        upd, _ = parareal(Gc, op, u0g, gpu_source(cfg), K, Uo, nsrc=1)
        torch.cuda.synchronize()
        res = oracle_parareal(op_o, truncs, u0, cfg.N, K, G.source_1d(cfg))
        got = Uo.cpu().numpy().T                       # (N+1, n)
        ref = res.U[K][:, 0]
        scale = np.max(np.linalg.norm(ref, axis=1))
        assert np.max(np.linalg.norm(got - ref, axis=1)) <= TAU_1D * scale, K


# ------------------------------------------- mass-matrix inner product (row 2)
def test_weighted_view_build_and_parareal_match_oracle():
    """pr_build_coarse / pr_parareal on the weighted view = the paper's method
    in the M inner product (generalized SVD): sigma and G_q' (in
    physical coordinates, G' x = C^{-1} G^' C x) against the oracle's weighted
    rSVD, and the Parareal iterates mapped back with C^{-1}."""
    import torch
    from paper_2508_08873_b200 import Coarse, parareal
    cfg = get("E2")
    base = gpu_op(cfg)
    view = base.weighted()
    Gg = Coarse.build(view, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    op_o = make_op(cfg)
    truncs = []
    for q in range(cfg.N):
        tr = rsvd_interval(op_o, q + 1, cfg.k, cfg.p, cfg.seed_omega, inner=op_o.M)
        truncs.append(tr)
        s1 = tr.sigma[0]
        assert np.max(np.abs(info["sigma"][q] - tr.sigma)) <= TAU_1D * s1, q
        X = np.random.default_rng(q).standard_normal((4, cfg.n))
        Xh = empty_batch(cfg, 4)
        view.to_weighted(to_gpu(cfg, X), Xh)
        Yh = empty_batch(cfg, 4)
        Gg.apply(q, Xh, Yh, 1)
        Y = empty_batch(cfg, 4)
        view.from_weighted(Yh, Y)
        got, ref = from_gpu(cfg, Y), tr.apply_linear(X)
        # the normwise bound holds in the M norm; in Euclidean norms it picks up
        # cond(C) = sqrt(cond(M)) <= sqrt(3) (P1 mass matrix): factor 2
        for v in range(4):
            assert np.linalg.norm(got[v] - ref[v]) <= 2 * TAU_1D * s1 * np.linalg.norm(X[v]), (q, v)
    u0 = G.initial_value(cfg)[None, :]
    u0g = torch.tensor(np.ascontiguousarray(u0.T), dtype=torch.float64, device="cuda")
    u0h = torch.zeros_like(u0g)
    view.to_weighted(u0g, u0h)
    for K in (0, 2):
        Uh = torch.zeros((cfg.n, cfg.N + 1), dtype=torch.float64, device="cuda")
        parareal(Gg, view, u0h, gpu_source(cfg), K, Uh, nsrc=1)
        U = torch.zeros_like(Uh)
        view.from_weighted(Uh, U)
        res = oracle_parareal(op_o, truncs, u0, cfg.N, K, G.source_1d(cfg))
        got = U.cpu().numpy().T
        ref = res.U[K][:, 0]
        scale = np.max(np.linalg.norm(ref, axis=1))
        assert np.max(np.linalg.norm(got - ref, axis=1)) <= TAU_1D * scale, K
