"""The interval-sharded path of the C ABI (include/pr.h "distribution") on one
GPU with in-process virtual ranks (pr_comm_create_local): P host
threads, each with its own stream, call pr_build_coarse(..., comm) and
pr_parareal collectively.  The result must be bit-identical to the unsharded
call -- coarse operators, delta / eps (all-reduced), every boundary state,
the update norms and ||b_n|| -- for P = 2, 3 (uneven shards) and 4.  This runs
the C++ schedule itself (halo sends, all-gathers of the reduced sweep data,
the first sweep matrix from the neighbour's U), not a model of it; only the
transport differs from NCCL (device copies ordered by events instead of NVLink
messages), and no kernel waits for another rank."""
import threading

import numpy as np
import pytest

from gpu_util import from_gpu, gpu_op, gpu_source, to_gpu
from workloads import generators as G
from workloads.configs import get

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    from paper_2508_08873_b200 import build as B
    B.build()
    assert torch.cuda.is_available()


def _batch(cfg, nvec):
    """Op-layout batch with a leading dimension padded to a multiple of 8 (the
    same alignment class for every shard, so the same kernel variants run)."""
    import torch
    if cfg.dim == 1:
        ld = (nvec + 7) // 8 * 8
        return torch.zeros((cfg.n, ld), dtype=torch.float64, device="cuda")[:, :nvec]
    P = cfg.n + 1
    return torch.zeros((nvec, P * P), dtype=torch.float64, device="cuda")


def _run(cfg, world):
    """Per rank: (first, n_local, info, u^K of its boundaries 1..nq, upd, bnorm)."""
    import torch
    from paper_2508_08873_b200 import Coarse, Comm, parareal
    op, src = gpu_op(cfg), gpu_source(cfg)
    S = cfg.nsrc if cfg.dim == 1 else 1
    u0 = np.stack([G.initial_value(cfg)] * S)
    u0g = to_gpu(cfg, u0)
    torch.cuda.synchronize()
    comms = Comm.local(world) if world > 1 else [None]
    out, errs = [None] * world, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega, comm=comms[r], stream=st)
                info = Gc.info()
                nq = info["n_local"]
                U = _batch(cfg, (nq + 1) * S)
                upd, bn = parareal(Gc, op, u0g if r == 0 else None, src, cfg.K, U, nsrc=S, stream=st)
                st.synchronize()
                got = from_gpu(cfg, U, (nq + 1) * S)[S:]
                out[r] = (info["first_interval"], nq, info, got, upd, bn)
                Gc.close()
        except Exception as e:                     # surfaced below (peers may then hang: test timeout)
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name", ["T4", "T4N", "C1", "T2D"])
def test_virtual_shards_bit_identical_to_unsharded(name):
    cfg = get(name)
    ref = _run(cfg, 1)[0]
    _, N, info1, u1, upd1, bn1 = ref
    for world in (2, 3, 4):
        parts = _run(cfg, world)
        starts = [p[0] for p in parts]
        assert starts[0] == 0 and sum(p[1] for p in parts) == cfg.N
        u = np.concatenate([p[3] for p in parts])
        np.testing.assert_array_equal(u, u1)
        sig = np.concatenate([p[2]["sigma"] for p in parts])
        np.testing.assert_array_equal(sig, info1["sigma"])
        for p in parts:
            assert p[2]["delta"] == info1["delta"] and p[2]["eps"] == info1["eps"]
            np.testing.assert_array_equal(p[4], upd1)
            np.testing.assert_array_equal(p[5], bn1)
