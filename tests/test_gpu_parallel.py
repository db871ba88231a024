"""The distributed building blocks of the C ABI (pr_coarse_project /
pr_reduced_sweep / pr_coarse_expand / pr_coarse_sweep_matrices / export)
driven by the interval-sharded orchestrator reproduce the monolithic
pr_parareal on one GPU (world size 1; several ranks on one GPU would run
NCCL kernels that wait on each other, so the multi-rank schedule is tested
on CPU with gloo in tests/test_parallel.py)."""
import numpy as np
import pytest

from gpu_util import empty_batch, from_gpu, gpu_op, gpu_source, to_gpu
from workloads import generators as G
from workloads.configs import get

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["T4", "T2D", "C1"])
def test_sharded_orchestrator_equals_pr_parareal(name):
    import torch
    from paper_2508_08873_b200 import Coarse, parareal
    from paper_2508_08873_b200.parallel import Blocks, Comm, LibprBackend, parareal_sharded
    cfg = get(name)
    op = gpu_op(cfg)
    src = gpu_source(cfg)
    S = cfg.nsrc
    u0 = np.stack([G.initial_value(cfg)] * S)
    u0g = to_gpu(cfg, u0)
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    Uo = empty_batch(cfg, (cfg.N + 1) * S)
    upd_ref, _ = parareal(Gc, op, u0g, src, cfg.K, Uo, nsrc=S)
    be = LibprBackend(op, Gc, cfg.N, 0, cfg.N, cfg.m, cfg.k, S, src)
    u, upd = parareal_sharded(be, Blocks(cfg.dim, op.rows, S, torch.device("cuda")), u0g, cfg.K, Comm())
    torch.cuda.synchronize()
    a, b = from_gpu(cfg, Uo), from_gpu(cfg, u)
    scale = np.max(np.abs(a))
    assert np.max(np.abs(a - b)) <= 1e-13 * scale
    np.testing.assert_allclose(upd.cpu().numpy(), upd_ref[:, 1:, :], rtol=1e-12, atol=1e-14 * scale)
