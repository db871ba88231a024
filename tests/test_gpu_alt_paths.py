"""The alternate kernels behind libpr's diagnostic switches (DESIGN.md
"Diagnostic switches") still match the oracle.  Each switch replaces one
kernel of the default path by its simpler fallback:

  PR_NO_PART        fused LU/UL streaming stepper (K1) instead of K1P
  PR_NO_SRC_BASIS   offsets b_n with the full source per source instead of the
                    source-basis combination
  PR_NO_XTY_RM      CUDA-core cross products instead of the row-major DMMA Gram
  PR_NO_TRSM_DMMA   row-wise substitution instead of the blocked DMMA TRSM
  PR_NO_RINV_CM     generic R^{-1} apply instead of the column-major DMMA one (2D)
  PR_NO_EXPAND_MMA  CUDA-core lift / reconstruction instead of the DMMA ones
  PR_PART_NOTMEM    K1P with every coefficient in shared memory (no tensor memory)
  PR_PART_NODM      K1P (tensor-memory variant, K = 16) with the banded interface
                    solve on the solver warps instead of the FP64 tensor-core product

A whole rSVD build + Parareal run (T4 in 1D, T2D in 2D) goes through the
switched kernel and is compared with the oracle at
the north-star tolerances.
"""
import functools

import numpy as np
import pytest

from gpu_util import TAU_1D, TAU_2D, empty_batch, from_gpu, gpu_op, gpu_source, to_gpu
from oracle.fine import make_op
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


@functools.lru_cache(maxsize=None)
def _oracle(name):
    cfg = get(name)
    op_o = make_op(cfg)
    truncs = [rsvd_interval(op_o, n, cfg.k, cfg.p, cfg.seed_omega) for n in range(1, cfg.N + 1)]
    S = cfg.nsrc
    if cfg.dim == 1:
        u0 = np.stack([G.initial_value(cfg)] * S)
        res = oracle_parareal(op_o, truncs, u0, cfg.N, cfg.K, G.source_1d(cfg), np.arange(S))
    else:
        u0 = G.initial_value(cfg)[None]
        res = oracle_parareal(op_o, truncs, u0, cfg.N, cfg.K, G.source_2d(cfg))
    return np.stack([t.sigma for t in truncs]), res, u0


def _run(name):
    from paper_2508_08873_b200 import Coarse, parareal
    cfg = get(name)
    opg = gpu_op(cfg)
    Gg = Coarse.build(opg, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gg.info()
    sig, res, u0 = _oracle(name)
    S = cfg.nsrc if cfg.dim == 1 else 1
    Uo = empty_batch(cfg, (cfg.N + 1) * S)
    upd, bn = parareal(Gg, opg, to_gpu(cfg, u0), gpu_source(cfg), cfg.K, Uo, nsrc=S)
    tau = TAU_1D if cfg.dim == 1 else TAU_2D
    assert np.max(np.abs(info["sigma"] - sig)) <= tau * sig.max()
    got = from_gpu(cfg, Uo).reshape((cfg.N + 1, S) + res.U.shape[3:])
    scale = np.max(np.abs(res.U))
    assert np.max(np.abs(got - res.U[cfg.K])) <= tau * scale


SWITCHES = ["PR_NO_PART", "PR_NO_SRC_BASIS", "PR_NO_XTY_RM", "PR_NO_TRSM_DMMA", "PR_NO_RINV_CM",
            "PR_NO_EXPAND_MMA", "PR_PART_VPT2"]


@pytest.mark.parametrize("switch", SWITCHES)
@pytest.mark.parametrize("name", ["T4", "T2D"])
def test_alternate_kernel_matches_oracle(name, switch, pr_env):
    if switch in ("PR_NO_PART", "PR_NO_SRC_BASIS", "PR_PART_VPT2") and name == "T2D":
        pytest.skip(f"{switch} concerns the 1D path only")
    pr_env(**{switch: "1"})
    _run(name)


@pytest.mark.parametrize("mode", ["linear", "adjoint", "affine"])
def test_two_vectors_per_lane_layout_at_c4_size(mode, pr_env):
    """PR_PART_VPT2: K1P with 32-row chunks and two vectors per lane (n > 8192)
    against the oracle's Thomas steps at C4's full grid (non-symmetric C4N)."""
    from gpu_util import relnorm
    from oracle.fine import fine
    from paper_2508_08873_b200 import PR_ADJOINT, PR_AFFINE, PR_LINEAR
    pr_env(PR_PART_VPT2="1")
    cfg = get("C4N")
    op_o, op_g = make_op(cfg), gpu_op(cfg)
    S = 4
    X = np.random.default_rng(3).standard_normal((2 * S, cfg.n))
    out = empty_batch(cfg, 2 * S)
    if mode == "affine":
        from dataclasses import replace
        cfg_s = replace(cfg, nsrc=S)
        op_g.fine_propagate(PR_AFFINE, 5, cfg.m, to_gpu(cfg, X), out, vecs_per_interval=S,
                            source=gpu_source(cfg_s))
        src = G.source_1d(cfg_s)
        ref = np.concatenate([fine(op_o, 6 + j, X[j * S:(j + 1) * S], "affine", src, np.arange(S))
                              for j in range(2)])
    else:
        op_g.fine_propagate(PR_LINEAR if mode == "linear" else PR_ADJOINT, 5, cfg.m, to_gpu(cfg, X), out)
        ref = fine(op_o, 6, X, mode)
    got = from_gpu(cfg, out)
    for v in range(2 * S):
        assert relnorm(got[v], ref[v]) <= TAU_1D


@pytest.mark.parametrize("switch", ["PR_PART_NOTMEM", "PR_PART_NODM"])
@pytest.mark.parametrize("mode", ["linear", "adjoint", "affine"])
def test_part_interface_variants_at_c4_size(mode, switch, pr_env):
    """K1P's alternate coefficient store / interface solve at C4's full grid
    (non-symmetric C4N: K = 16 chunks per CTA, the shape the tensor-memory and
    tensor-core variants serve) against the oracle's Thomas steps."""
    from gpu_util import relnorm
    from oracle.fine import fine
    from paper_2508_08873_b200 import PR_ADJOINT, PR_AFFINE, PR_LINEAR
    pr_env(**{switch: "1"})
    cfg = get("C4N")
    op_o, op_g = make_op(cfg), gpu_op(cfg)
    S = 4
    X = np.random.default_rng(5).standard_normal((2 * S, cfg.n))
    out = empty_batch(cfg, 2 * S)
    if mode == "affine":
        from dataclasses import replace
        cfg_s = replace(cfg, nsrc=S)
        op_g.fine_propagate(PR_AFFINE, 5, cfg.m, to_gpu(cfg, X), out, vecs_per_interval=S,
                            source=gpu_source(cfg_s))
        src = G.source_1d(cfg_s)
        ref = np.concatenate([fine(op_o, 6 + j, X[j * S:(j + 1) * S], "affine", src, np.arange(S))
                              for j in range(2)])
    else:
        op_g.fine_propagate(PR_LINEAR if mode == "linear" else PR_ADJOINT, 5, cfg.m, to_gpu(cfg, X), out)
        ref = fine(op_o, 6, X, mode)
    got = from_gpu(cfg, out)
    for v in range(2 * S):
        assert relnorm(got[v], ref[v]) <= TAU_1D
