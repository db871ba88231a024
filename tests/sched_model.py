"""Executable model of libpr's interval-sharded Parareal schedule (the C++ in
pr_api.cu `pr_parareal` with a communicator), written
with torch.distributed collectives so the exchange pattern runs on CPU with
gloo (tests/test_parallel.py).  The GPU tests check that the C++ schedule
gives bit-identical results across world sizes with in-process virtual ranks
(tests/test_gpu_parallel.py).

Rank r owns the contiguous intervals q0 .. q0+nq-1 (shard()).  Arrays hold
nq+1 "blocks" of S vectors; block i is boundary q0+i, block 0 the halo (the
left neighbour's last block, u0 on rank 0).  One iteration (eq.
def_Parareal) in reduced coordinates:
  1. fine solves of the local intervals        Fu_{q+1} = F'_q u_q + b_q
  2. halo: the left neighbour's last Fu block   -> Fu_{q0}
  3. local projections                          d_q = Sigma_q V_q^T (Fu_q - u_q)
  4. all-gather of d; every rank runs the k-dimensional sweep
     e_q = C_q e_{q-1} + d_q over all N intervals
  5. local reconstruction + update norms        u_{q+1} = Fu_{q+1} + U_q e_q
  6. halo: the left neighbour's last u block    -> u_{q0}
"""
from __future__ import annotations

import torch

from paper_2508_08873_b200.parallel import shard


class TorchComm:
    """torch.distributed stand-in for pr_comm (world == 1 needs no process group)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.on = dist.is_available() and dist.is_initialized()
        self.group = group
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1

    def shift_right(self, t):
        """Send t to rank+1; return what rank-1 sent (None on rank 0)."""
        if self.world == 1:
            return None
        dist = self.dist
        t = t.contiguous()
        recv = torch.empty_like(t) if self.rank > 0 else None
        ops = []
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, t, self.rank + 1, self.group))
        if self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, recv, self.rank - 1, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return recv

    def all_gather_v(self, t, counts):
        """Concatenation of every rank's t (counts[r] rows) along dim 0: padded
        to max(counts) rows for the collective, then compacted (pr_comm.cu
        all_gather_v does the same)."""
        if self.world == 1:
            return t
        mx = max(counts)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


class Blocks:
    """Block arrays in the op layout: 1D (rows, nblocks*S), 2D (nblocks*S, rows)."""

    def __init__(self, dim: int, rows: int, S: int, device, dtype=torch.float64):
        self.dim, self.rows, self.S, self.device, self.dtype = dim, rows, S, device, dtype

    def new(self, nblocks: int):
        shape = (self.rows, nblocks * self.S) if self.dim == 1 else (nblocks * self.S, self.rows)
        return torch.zeros(shape, dtype=self.dtype, device=self.device)

    def view(self, t, i0: int, i1: int):
        S = self.S
        return t[:, i0 * S:i1 * S] if self.dim == 1 else t[i0 * S:i1 * S]


def parareal_sharded(backend, blocks: Blocks, u0, K: int, comm: TorchComm):
    """K Parareal iterations on this rank's intervals (backend: stage
    implementation for intervals [backend.q0, backend.q0 + backend.nq)).
    Returns (u, upd): u holds blocks q0 .. q0+nq; upd (K, N, S)."""
    nq, N, S = backend.nq, backend.N, backend.S
    q0 = backend.q0
    counts = [shard(N, r, comm.world)[1] for r in range(comm.world)]
    u, Fu, b = blocks.new(nq + 1), blocks.new(nq + 1), blocks.new(nq)
    backend.offsets(b)
    blocks.view(Fu, 1, nq + 1).copy_(b)
    U_prev = comm.shift_right(backend.last_U())
    C_all = comm.all_gather_v(backend.local_C(U_prev), counts)

    def halo(arr):
        got = comm.shift_right(blocks.view(arr, nq, nq + 1).contiguous())
        blocks.view(arr, 0, 1).copy_(u0 if comm.rank == 0 else got)

    d = backend.new_d(nq)
    e_all = backend.new_d(N)
    halo(Fu)
    backend.project(None, blocks.view(Fu, 0, nq), d)
    backend.sweep(C_all, comm.all_gather_v(d, counts), e_all)
    backend.expand(blocks.view(Fu, 1, nq + 1), e_all[q0:q0 + nq], blocks.view(u, 1, nq + 1), None)
    halo(u)
    upd = []
    for _ in range(K):
        backend.fine(blocks.view(u, 0, nq), blocks.view(Fu, 1, nq + 1), b)
        halo(Fu)
        backend.project(blocks.view(u, 0, nq), blocks.view(Fu, 0, nq), d)
        backend.sweep(C_all, comm.all_gather_v(d, counts), e_all)
        un = backend.new_norms(nq)
        backend.expand(blocks.view(Fu, 1, nq + 1), e_all[q0:q0 + nq], blocks.view(u, 1, nq + 1), un)
        halo(u)
        upd.append(comm.all_gather_v(un, counts))
    upd = torch.stack(upd).reshape(K, N, S) if K > 0 else torch.zeros((0, N, S))
    return u, upd
