"""GPU parity of the 1D CUDA path against the oracle (same seeded inputs),
through the C ABI.  Tolerances: BASELINE.json north_star, 1e-10 normwise for
fp64 states and singular values (reading Z11)."""
from dataclasses import replace

import numpy as np
import pytest

from gpu_util import TAU_1D, empty_batch, from_gpu, gpu_op, gpu_source, relnorm, to_gpu
from oracle.fine import fine, make_op, sequential_reference
from oracle.parareal import parareal as oracle_parareal
from oracle.rng import gaussian_sketch
from oracle.rsvd import rsvd_interval
from workloads import generators as G
from workloads.configs import C1, C2, C4, get

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    from paper_2508_08873_b200 import build as B
    B.build()
    assert torch.cuda.is_available()


# ------------------------------------------------------------------ sketch
@pytest.mark.parametrize("n,nint,l,q0", [(127, 3, 12, 0), (301, 2, 7, 5), (1001, 1, 40, 63)])
def test_gaussian_sketch_matches_oracle(n, nint, l, q0):
    cfg = replace(C1, n=n)
    op = gpu_op(cfg)
    out = empty_batch(cfg, nint * l)
    op.gaussian_sketch(q0, nint, l, 2508088730, out)
    got = out.cpu().numpy()
    for j in range(nint):
        ref = gaussian_sketch(2508088730, q0 + j, n, l)
        # counter-based: identical integers, Box-Muller to a few ulps
        np.testing.assert_allclose(got[:, j * l:(j + 1) * l], ref, rtol=0, atol=1e-14)


# -------------------------------------------------------------- fine solver
def _stepper_path(pr_env, path):
    """Select the 1D stepper: the fused one-vector-per-thread kernel (K1) or the
    cluster-partitioned kernel (K1P, k_part.cu; the default for every n it
    supports)."""
    pr_env(PR_NO_PART="1" if path == "fused" else None)


@pytest.mark.parametrize("name,n,m,B", [("C1", 127, 64, 12), ("C1", 127, 1, 6), ("C1", 127, 2, 5),
                                        ("T4", 301, 16, 33), ("T4", 37, 7, 64), ("T1", 200, 12, 70),
                                        ("C1", 64, 5, 33), ("C2", 513, 7, 9), ("C4", 16384, 3, 17),
                                        ("C2", 4095, 256, 10), ("C2", 8192, 20, 3),
                                        ("C4", 16383, 128, 6),
                                        # non-symmetric A: F'^* is a different map
                                        ("T4N", 301, 16, 33), ("C4N", 4095, 64, 9),
                                        ("C4N", 16383, 128, 6)])
@pytest.mark.parametrize("mode", ["linear", "adjoint"])
@pytest.mark.parametrize("path", ["fused", "part"])
def test_fine_linear_adjoint(name, n, m, B, mode, path, pr_env):
    _stepper_path(pr_env, path)
    from paper_2508_08873_b200 import PR_ADJOINT, PR_LINEAR
    cfg = replace(get(name), n=n, m=m)
    op_o = make_op(cfg)
    op_g = gpu_op(cfg)
    rng = np.random.default_rng(n + m + B)
    X = rng.standard_normal((B, n))
    Ug = to_gpu(cfg, X)
    out = empty_batch(cfg, B)
    op_g.fine_propagate(PR_LINEAR if mode == "linear" else PR_ADJOINT, 2, m, Ug, out)
    ref = fine(op_o, 3, X, mode)
    got = from_gpu(cfg, out)
    for v in range(B):
        assert relnorm(got[v], ref[v]) <= TAU_1D, v


@pytest.mark.parametrize("name,B,ld", [("T4", 5 * 4, 20), ("T4", 5 * 3, 17), ("C1", 8, 8)])
@pytest.mark.parametrize("path", ["fused", "part"])
def test_fine_affine_offset_and_inplace(name, B, ld, path, pr_env):
    _stepper_path(pr_env, path)
    from paper_2508_08873_b200 import PR_AFFINE, PR_LINEAR
    cfg = get(name)
    op_o, op_g = make_op(cfg), gpu_op(cfg)
    src_g = gpu_source(cfg)
    src_o = G.source_1d(cfg)
    S = cfg.nsrc
    nint = B // S
    rng = np.random.default_rng(B)
    X = rng.standard_normal((B, cfg.n))
    Ug = to_gpu(cfg, X, ld)
    out = empty_batch(cfg, B, ld)
    q0 = 1
    op_g.fine_propagate(PR_AFFINE, q0, cfg.m, Ug, out, vecs_per_interval=S, source=src_g)
    got = from_gpu(cfg, out, B)
    ref = np.zeros_like(X)
    for j in range(nint):
        sl = slice(j * S, (j + 1) * S)
        ref[sl] = fine(op_o, q0 + j + 1, X[sl], "affine", src_o, np.arange(S))
    for v in range(B):
        assert relnorm(got[v], ref[v]) <= TAU_1D
    # zero input == offsets b_q; then F'u + b via the offset path, in place
    b = empty_batch(cfg, B, ld)
    op_g.fine_propagate(PR_AFFINE, q0, cfg.m, None, b, vecs_per_interval=S, source=src_g)
    op_g.fine_propagate(PR_LINEAR, q0, cfg.m, Ug, Ug, offset=b)
    got2 = from_gpu(cfg, Ug, B)
    for v in range(B):
        assert relnorm(got2[v], ref[v]) <= TAU_1D


def test_fine_m0_is_copy():
    from paper_2508_08873_b200 import PR_LINEAR
    cfg = C1
    op_g = gpu_op(cfg)
    X = np.random.default_rng(0).standard_normal((9, cfg.n))
    out = empty_batch(cfg, 9)
    op_g.fine_propagate(PR_LINEAR, 0, 0, to_gpu(cfg, X), out)
    np.testing.assert_array_equal(from_gpu(cfg, out), X)


# ------------------------------------------------------------------- build
def _check_interval(cfg, Gg, q, info, probes=6):
    """G_q' of the GPU vs the oracle's rSVD of the same interval (operator
    norm on Gaussian probes, and sigma normwise)."""
    import torch
    op_o = make_op(cfg)
    tr = rsvd_interval(op_o, q + 1, cfg.k, cfg.p, cfg.seed_omega)
    s1 = tr.sigma[0]
    assert np.max(np.abs(info["sigma"][q] - tr.sigma)) <= TAU_1D * s1
    X = np.random.default_rng(q).standard_normal((probes, cfg.n))
    Y = empty_batch(cfg, probes)
    Gg.apply(q, to_gpu(cfg, X), Y, 1)
    got = from_gpu(cfg, Y)
    ref = tr.apply_linear(X)
    for v in range(probes):
        assert np.linalg.norm(got[v] - ref[v]) <= TAU_1D * s1 * np.linalg.norm(X[v])


@pytest.mark.parametrize("name", ["C4N", "T4N"])
def test_adjoint_differs_from_forward_nonsymmetric(name):
    """On the convection-diffusion operator F'^* != F' (by ~beta h / kappa),
    so the adjoint parity above would catch a forward/transpose mix-up."""
    from paper_2508_08873_b200 import PR_ADJOINT, PR_LINEAR
    cfg = get(name)
    op_g = gpu_op(cfg)
    X = np.random.default_rng(5).standard_normal((4, cfg.n))
    a, b = empty_batch(cfg, 4), empty_batch(cfg, 4)
    op_g.fine_propagate(PR_LINEAR, 0, cfg.m, to_gpu(cfg, X), a)
    op_g.fine_propagate(PR_ADJOINT, 0, cfg.m, to_gpu(cfg, X), b)
    fa, fb = from_gpu(cfg, a), from_gpu(cfg, b)
    for v in range(4):
        assert relnorm(fa[v], fb[v]) > 1e-6


@pytest.mark.parametrize("name", ["C1", "T1", "T1k1", "T4", "T4N"])
def test_build_all_intervals(name):
    from paper_2508_08873_b200 import Coarse
    cfg = get(name)
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    for q in range(cfg.N):
        _check_interval(cfg, Gg, q, info)
    sig = info["sigma"]
    assert info["delta"] == np.max(sig[:, 0])
    assert info["eps"] == np.max(sig[:, cfg.k])


@pytest.mark.parametrize("name,qs", [("C2", (0, 31, 63)), ("C4", (0, 255)), ("C4N", (0, 255))])
def test_build_full_size_sampled_intervals(name, qs):
    from paper_2508_08873_b200 import Coarse
    cfg = get(name)
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    for q in qs:
        _check_interval(cfg, Gg, q, info)


def test_build_sharded_equals_full():
    """Seeds depend on (seed, q, column) only: building intervals [3, 7) alone
    gives the same coarse operators as building all of them (S:495 analog)."""
    from paper_2508_08873_b200 import Coarse
    cfg = get("T1")
    opg = gpu_op(cfg)
    full = Coarse.build(opg, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega).info()
    part = Coarse.build(opg, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega, first_interval=3,
                        n_local=4).info()
    np.testing.assert_array_equal(part["sigma"], full["sigma"][3:7])


# ---------------------------------------------------------------- Parareal
def _run_parareal(cfg, K=None, keep_hist=True):
    import torch
    from paper_2508_08873_b200 import Coarse, parareal
    K = cfg.K if K is None else K
    opg = gpu_op(cfg)
    Gg = Coarse.build(opg, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    S = cfg.nsrc
    u0 = np.stack([G.initial_value(cfg)] * S)
    u0g = to_gpu(cfg, u0)
    nvec = (cfg.N + 1) * S
    Uo = empty_batch(cfg, nvec)
    hist = None
    if keep_hist:
        hist = torch.zeros((K + 1,) + tuple(Uo.shape), dtype=torch.float64, device="cuda")
    upd, bn = parareal(Gg, opg, u0g, gpu_source(cfg), K, Uo, nsrc=S, hist=hist)
    return Gg, info, Uo, hist, upd, bn, u0


@pytest.mark.parametrize("name", ["T1", "T4", "T1k1", "C1", "T4N", "T4S"])
def test_parareal_all_iterates_match_oracle(name):
    cfg = get(name)
    Gg, info, Uo, hist, upd, bn, u0 = _run_parareal(cfg)
    op_o = make_op(cfg)
    truncs = [rsvd_interval(op_o, n, cfg.k, cfg.p, cfg.seed_omega) for n in range(1, cfg.N + 1)]
    S = cfg.nsrc
    res = oracle_parareal(op_o, truncs, u0, cfg.N, cfg.K, G.source_1d(cfg), np.arange(S))
    scale = np.max(np.linalg.norm(res.U, axis=-1))
    for k in range(cfg.K + 1):
        got = from_gpu(cfg, hist[k]).reshape(cfg.N + 1, S, cfg.n)
        err = np.max(np.linalg.norm(got - res.U[k], axis=-1))
        assert err <= TAU_1D * scale, (k, err / scale)
    # update norms ||u^k_n - u^{k-1}_n|| and offsets ||b_n|| (b_0 = u0)
    assert np.max(np.abs(upd - res.upd[1:])) <= TAU_1D * scale
    bref = np.linalg.norm(res.b, axis=-1)
    bref[0] = np.linalg.norm(u0, axis=-1)
    assert np.max(np.abs(bn - bref)) <= TAU_1D * np.max(bref)
    np.testing.assert_array_equal(upd[:, 0], 0.0)


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_parareal_full_size_against_fine_solution(name):
    """At full size the Parareal fixed point is the sequential fine solution
    (P:136-139): compare sampled sources with the oracle's
    sequential propagation, and finite termination u^k_n = u_n for n <= k."""
    cfg = get(name)
    Gg, info, Uo, hist, upd, bn, u0 = _run_parareal(cfg, keep_hist=False)
    S = cfg.nsrc
    sample = [0, S - 1] if S > 1 else [0]
    op_o = make_op(cfg)
    src = G.source_1d(cfg)
    ref = sequential_reference(op_o, u0[sample], cfg.N, src, np.array(sample))
    got = from_gpu(cfg, Uo).reshape(cfg.N + 1, S, cfg.n)[:, sample]
    scale = np.max(np.linalg.norm(ref, axis=-1))
    err = np.max(np.linalg.norm(got - ref, axis=-1))
    assert err <= TAU_1D * scale, err / scale


@pytest.mark.parametrize("name", ["C1", "T4", "C4"])
def test_lifted_factors_orthonormal_and_deterministic(name):
    """U_q = W Psi_k and V_q = V Phi_k have orthonormal columns (steps 2, 4, 5
    of P:258-299 produce orthonormal bases; Psi, Phi orthogonal), and a rebuild
    with the same seed is bit-identical (counter-based sketch, fixed-order
    reductions)."""
    import torch
    from paper_2508_08873_b200 import Coarse
    cfg = get(name)
    op = gpu_op(cfg)
    G1 = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    G2 = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    i1, i2 = G1.info(), G2.info()
    np.testing.assert_array_equal(i1["sigma"], i2["sigma"])
    U = torch.empty((op.rows, cfg.k), dtype=torch.float64, device="cuda")
    V = torch.empty_like(U)
    U2, V2 = torch.empty_like(U), torch.empty_like(U)
    I = torch.eye(cfg.k, dtype=torch.float64, device="cuda")
    for q in sorted({0, cfg.N // 2, cfg.N - 1}):
        G1.export_interval(q, U_q=U, V_q=V)
        G2.export_interval(q, U_q=U2, V_q=V2)
        assert float((U.T @ U - I).abs().max()) < 1e-13
        assert float((V.T @ V - I).abs().max()) < 1e-13
        assert torch.equal(U, U2) and torch.equal(V, V2)


def _core_amplification(op_o, cfg, qi, q):
    """||Psi||_2 ||(Psi^T W)^{-1}||_2 of the independent-adjoint core solve
    C = (Psi^T W)^{-1} Z^T V (reading R-IND): a perturbation dZ of
    the adjoint sketch (rounding of two differently ordered fp64 steppers,
    ~tau ||F'|| ||Psi||) moves C by up to this factor times tau ||F'||, so
    the normwise sigma tolerance of this variant is tau sigma_1 times it."""
    from oracle.linalg import householder_qr
    l = cfg.k + cfg.p
    Om = gaussian_sketch(cfg.seed_omega, qi, cfg.n, l)
    Y = fine(op_o, qi + 1, Om.T, "linear").T
    for _ in range(q):
        Qz, _ = householder_qr(fine(op_o, qi + 1, householder_qr(Y)[0].T, "adjoint").T)
        Y = fine(op_o, qi + 1, Qz.T, "linear").T
    W, _ = householder_qr(Y)
    Psi = gaussian_sketch(cfg.seed_omega, qi, cfg.n, l, stream=2)
    return np.linalg.norm(Psi, 2) / np.linalg.svd(Psi.T @ W, compute_uv=False)[-1]


@pytest.mark.parametrize("q,indep", [(1, False), (0, True), (2, True)])
@pytest.mark.parametrize("name", ["C1", "T4", "T4N"])
def test_build_rsvd_variants_match_oracle(name, q, indep):
    """Power iterations and the independent adjoint sketch
    (P:335-337): every interval's sigma and G_q' against the oracle's variant."""
    from paper_2508_08873_b200 import Coarse
    cfg = get(name)
    Gg = Coarse.build(gpu_op(cfg), cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega, power_iterations=q,
                      independent_adjoint=indep)
    info = Gg.info()
    op_o = make_op(cfg)
    for qi in range(cfg.N):
        tr = rsvd_interval(op_o, qi + 1, cfg.k, cfg.p, cfg.seed_omega, power_iterations=q,
                           independent_adjoint=indep)
        s1 = tr.sigma[0] * (_core_amplification(op_o, cfg, qi, q) if indep else 1.0)
        assert np.max(np.abs(info["sigma"][qi] - tr.sigma)) <= TAU_1D * s1, qi
        X = np.random.default_rng(qi).standard_normal((4, cfg.n))
        Y = empty_batch(cfg, 4)
        Gg.apply(qi, to_gpu(cfg, X), Y, 1)
        got, ref = from_gpu(cfg, Y), tr.apply_linear(X)
        for v in range(4):
            assert np.linalg.norm(got[v] - ref[v]) <= TAU_1D * s1 * np.linalg.norm(X[v]), (qi, v)


# ---------------------------------------------------- race detector by repetition
@pytest.mark.parametrize("name,B,env", [("C2", 64, None), ("C2", 2560, None), ("C4", 1024, None),
                                        ("C4", 1024, "PR_PART_VPT2"), ("T4", 40, None)])
def test_part_stepper_bitwise_repeatable(name, B, env, monkeypatch):
    """compute-sanitizer is not available on the GPU pool; a race in K1P's
    shared-memory / DSMEM / mbarrier hand-offs would show up as run-to-run
    differences.  20 identical launches (LINEAR and ADJOINT) must agree bit for
    bit (H = 1 and H = 2 chunk layouts, the two-vectors-per-lane layout)."""
    import torch
    from paper_2508_08873_b200 import PR_ADJOINT, PR_LINEAR, lib
    if env:
        monkeypatch.setenv(env, "1")
    lib().pr_reload_env()
    try:
        cfg = get(name)
        op = gpu_op(cfg)
        X = torch.randn(cfg.n, B, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
        for mode in (PR_LINEAR, PR_ADJOINT):
            Y0 = torch.empty_like(X)
            op.fine_propagate(mode, 0, cfg.m, X, Y0)
            for _ in range(20):
                Y = torch.empty_like(X)
                op.fine_propagate(mode, 0, cfg.m, X, Y)
                assert torch.equal(Y, Y0)
    finally:
        if env:
            monkeypatch.delenv(env)
        lib().pr_reload_env()


@pytest.mark.parametrize("name,n,m,B,ld", [("C4", 16383, 9, 341, 343),   # ragged last group, odd ld (8-byte staging)
                                           ("C4", 16383, 5, 1000, 1000),  # 16-byte staging
                                           ("C2", 4095, 7, 777, 778),
                                           ("T4", 301, 6, 1500, 1501)])
def test_part_persistent_clusters(name, n, m, B, ld, pr_env):
    """K1P runs as many clusters as are co-resident, each looping over vector
    groups with the next group's input staged in shared memory by cp.async
    (k_part.cu).  Batches of many groups per cluster, a ragged last group, odd
    and even leading dimensions, a stored offset and in-place operation must
    give the one-cluster-per-group launch bit for bit, and the oracle on
    sampled vectors."""
    import torch
    from paper_2508_08873_b200 import PR_ADJOINT, PR_LINEAR
    cfg = replace(get(name), n=n, m=m)
    op_g = gpu_op(cfg)
    op_o = make_op(cfg)
    rng = np.random.default_rng(B + ld)
    X = rng.standard_normal((B, n))
    Off = rng.standard_normal((B, n))
    res = {}
    for persist in (True, False):
        pr_env(PR_PART_NOPERSIST=None if persist else "1")
        for mode in (PR_LINEAR, PR_ADJOINT):
            Ug = to_gpu(cfg, X, ld)
            out = empty_batch(cfg, B, ld)
            op_g.fine_propagate(mode, 1, m, Ug, out, B=B)
            Og = to_gpu(cfg, Off, ld)
            op_g.fine_propagate(mode, 1, m, Ug, Ug, offset=Og, B=B)     # in place, + offset
            res[(persist, mode)] = (out.clone(), Ug.clone())
    for mode in (PR_LINEAR, PR_ADJOINT):
        a, b = res[(True, mode)], res[(False, mode)]
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), mode
    sample = np.unique(np.r_[0, 1, 15, 16, B // 2, B - 17, B - 2, B - 1])
    for mode, mname in ((PR_LINEAR, "linear"), (PR_ADJOINT, "adjoint")):
        ref = fine(op_o, 2, X[sample], mname)
        got = from_gpu(cfg, res[(True, mode)][0], B)[sample]
        got2 = from_gpu(cfg, res[(True, mode)][1], B)[sample]
        for i in range(len(sample)):
            assert relnorm(got[i], ref[i]) <= TAU_1D, (mname, sample[i])
            assert relnorm(got2[i], ref[i] + Off[sample[i]]) <= TAU_1D, (mname, sample[i])


def test_coarse_estimate_and_adaptive_p_match_oracle():
    """pr_coarse_estimate against the oracle's estimator on every interval, and
    pr_build_coarse_adaptive stopping at the p the estimates prescribe."""
    from paper_2508_08873_b200 import Coarse
    from oracle.rsvd import coarse_error_estimate
    cfg = get("T1")
    op = gpu_op(cfg)
    op_o = make_op(cfg)
    ests = {}
    for p in (1, 2, 4):
        Gg = Coarse.build(op, cfg.N, cfg.m, cfg.k, p, cfg.seed_omega)
        est = Gg.estimate(op, 10, cfg.seed_omega)
        ref = []
        for q in range(cfg.N):
            tr = rsvd_interval(op_o, q + 1, cfg.k, p, cfg.seed_omega)
            ref.append(coarse_error_estimate(op_o, tr, q + 1, 10, cfg.seed_omega))
            # probes have norm ~ sqrt(n); the estimate is a norm of F'w - G'w
            assert abs(est[q] - ref[-1]) <= TAU_1D * tr.sigma[0] * 20 * np.sqrt(cfg.n), (p, q)
        ests[p] = max(ref)
    # a tolerance between the p = 2 and the p = 1 estimates: doubling stops at p = 2
    if ests[2] < ests[1]:
        tol = np.sqrt(ests[1] * ests[2])
        Ga, pu = Coarse.build_adaptive(op, cfg.N, cfg.m, cfg.k, 1, 8, tol, cfg.seed_omega, r=10)
        assert pu == 2
        assert Ga.info()["l"] == cfg.k + 2
