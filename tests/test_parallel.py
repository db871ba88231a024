"""Multi-process (gloo, CPU) tests of the interval-sharded schedule: the
executable model of libpr's sharded pr_parareal (tests/sched_model.py) must
give bit-identical results for world sizes 1, 2, 3 (uneven shards) and 4, and
agree with the oracle's direct Parareal.  The stages run on a
test-only numpy backend with the semantics of the CUDA library's stages.  Also
the communicator bootstrap of paper_2508_08873_b200/parallel.py (NCCL unique
id made on rank 0 and broadcast) with a host-only stand-in for the library."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle.fine import fine, make_op
from oracle.parareal import parareal as oracle_parareal
from oracle.rsvd import rsvd_interval
from paper_2508_08873_b200.parallel import nccl_comm, shard
from sched_model import Blocks, TorchComm, parareal_sharded
from workloads import generators as G
from workloads.configs import get

CFG = "T4"


class NumpyBackend:
    """CPU stand-in for LibprBackend (1D layout: block i = columns i*S..(i+1)*S)."""

    def __init__(self, cfg, truncs, q0, nq):
        self.cfg, self.truncs, self.q0, self.nq = cfg, truncs, q0, nq
        self.N, self.k, self.S = cfg.N, cfg.k, cfg.nsrc
        self.op = make_op(cfg)
        self.src = G.source_1d(cfg)

    def _blk(self, t, i):
        return t[:, i * self.S:(i + 1) * self.S]

    def new_d(self, nint):
        return torch.zeros((nint, self.k, self.S), dtype=torch.float64)

    def new_norms(self, nint):
        return torch.zeros((nint, self.S), dtype=torch.float64)

    def offsets(self, out):
        z = np.zeros((self.S, self.cfg.n))
        for i in range(self.nq):
            b = fine(self.op, self.q0 + i + 1, z, "affine", self.src, np.arange(self.S))
            self._blk(out, i).copy_(torch.from_numpy(b.T))

    def fine(self, u_in, out, b):
        for i in range(self.nq):
            x = self._blk(u_in, i).numpy().T
            y = fine(self.op, self.q0 + i + 1, x, "linear")
            self._blk(out, i).copy_(torch.from_numpy(y.T) + self._blk(b, i))

    def last_U(self):
        return torch.from_numpy(self.truncs[self.q0 + self.nq - 1].U.copy())

    def local_C(self, U_prev):
        C = torch.zeros((self.nq, self.k, self.k), dtype=torch.float64)
        for i in range(self.nq):
            q = self.q0 + i
            tr = self.truncs[q]
            if i == 0:
                if U_prev is None:
                    continue
                Up = U_prev.numpy()
            else:
                Up = self.truncs[q - 1].U
            C[i] = torch.from_numpy(tr.sigma[: self.k, None] * (tr.V.T @ Up))
        return C

    def project(self, Y1, Y2, d):
        for i in range(self.nq):
            tr = self.truncs[self.q0 + i]
            y = self._blk(Y2, i).numpy() - (self._blk(Y1, i).numpy() if Y1 is not None else 0.0)
            d[i] = torch.from_numpy(tr.sigma[: self.k, None] * (tr.V.T @ y))

    def sweep(self, C_all, d_all, e_all):
        e = np.zeros((self.k, self.S))
        for j in range(self.N):
            e = (C_all[j].numpy() @ e if j > 0 else 0.0) + d_all[j].numpy()
            e_all[j] = torch.from_numpy(e)

    def expand(self, Fu, e_loc, out, upd):
        for i in range(self.nq):
            tr = self.truncs[self.q0 + i]
            new = self._blk(Fu, i).numpy() + tr.U @ e_loc[i].numpy()
            if upd is not None:
                upd[i] = torch.from_numpy(np.linalg.norm(new - self._blk(out, i).numpy(), axis=0))
            self._blk(out, i).copy_(torch.from_numpy(new))


def _setup():
    cfg = get(CFG)
    op = make_op(cfg)
    truncs = [rsvd_interval(op, n, cfg.k, cfg.p, cfg.seed_omega) for n in range(1, cfg.N + 1)]
    u0 = np.stack([G.initial_value(cfg)] * cfg.nsrc)
    return cfg, truncs, u0


def _run(rank, world, outdir, port):
    cfg, truncs, u0 = _setup()
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    comm = TorchComm()
    q0, nq = shard(cfg.N, comm.rank, comm.world)
    be = NumpyBackend(cfg, truncs, q0, nq)
    blocks = Blocks(1, cfg.n, cfg.nsrc, "cpu")
    u0b = torch.from_numpy(np.ascontiguousarray(u0.T))
    u, upd = parareal_sharded(be, blocks, u0b, cfg.K, comm)
    np.save(os.path.join(outdir, f"u_{world}_{rank}.npy"), u.numpy())
    np.save(os.path.join(outdir, f"upd_{world}_{rank}.npy"), upd.numpy())
    if world > 1:
        torch.distributed.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather(outdir, world, cfg):
    """Reassemble u^K_{1..N} (N, S, n) from the ranks' local blocks 1..nq."""
    parts, upd = [], None
    for r in range(world):
        u = np.load(os.path.join(outdir, f"u_{world}_{r}.npy"))
        q0, nq = shard(cfg.N, r, world)
        blocks = u[:, cfg.nsrc:].T.reshape(nq, cfg.nsrc, cfg.n)
        parts.append(blocks)
        upd = np.load(os.path.join(outdir, f"upd_{world}_{r}.npy"))
    return np.concatenate(parts), upd


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("par"))
    _run(0, 1, out, 0)
    for world in (2, 3, 4):
        torch.multiprocessing.spawn(_run, args=(world, out, _free_port()), nprocs=world, join=True)
    return out


def test_sharded_parareal_is_world_size_invariant(runs):
    cfg = get(CFG)
    u1, upd1 = _gather(runs, 1, cfg)
    for world in (2, 3, 4):
        uw, updw = _gather(runs, world, cfg)
        np.testing.assert_array_equal(uw, u1)
        np.testing.assert_array_equal(updw, upd1)


def test_sharded_parareal_matches_oracle_direct_form(runs):
    cfg, truncs, u0 = _setup()
    res = oracle_parareal(make_op(cfg), truncs, u0, cfg.N, cfg.K, G.source_1d(cfg),
                          np.arange(cfg.nsrc))
    u1, upd1 = _gather(runs, 1, cfg)
    scale = np.max(np.abs(res.U))
    assert np.max(np.abs(u1 - res.U[cfg.K, 1:])) <= 1e-12 * scale
    assert np.max(np.abs(upd1 - res.upd[1:, 1:])) <= 1e-12 * scale


def test_shard_partition():
    for total in (7, 16, 256):
        for world in (1, 2, 3, 8):
            spans = [shard(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == total
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1


class _FakeComm:
    """Host-only stand-in for paper_2508_08873_b200.Comm (no NCCL, no GPU)."""
    made = []

    @staticmethod
    def nccl_unique_id():
        return bytes(range(128))

    @classmethod
    def nccl(cls, rank, world, uid):
        return (rank, world, uid)


def _boot(rank, world, outdir, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    r, w, uid = nccl_comm(api=_FakeComm)
    np.save(os.path.join(outdir, f"boot_{rank}.npy"), np.frombuffer(uid, dtype=np.uint8))
    assert (r, w) == (rank, world)
    torch.distributed.destroy_process_group()


def test_nccl_bootstrap_broadcasts_rank0_id(tmp_path):
    """Every rank joins with rank 0's unique id (the other ranks never make one)."""
    world = 3
    torch.multiprocessing.spawn(_boot, args=(world, str(tmp_path), _free_port()), nprocs=world, join=True)
    for r in range(world):
        got = np.load(os.path.join(str(tmp_path), f"boot_{r}.npy"))
        np.testing.assert_array_equal(got, np.arange(128, dtype=np.uint8))
