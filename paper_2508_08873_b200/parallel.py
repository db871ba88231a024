"""Interval-sharded Parareal over several GPUs (one process per GPU).

Rank r owns the contiguous intervals q0 .. q0+nq-1 (paper intervals q+1).  Its
coarse solvers come from `pr_build_coarse(first_interval=q0, n_local=nq)` --
no communication (seeds depend only on (seed, q, column)).  One Parareal
iteration (eq. def_Parareal) in the reduced form of DESIGN.md §6:

  1. fine solves of the local intervals        Fu_{q+1} = F'_q u_q + b_q
  2. halo: the left neighbour's last Fu block   -> Fu_{q0}          (P2P, n*S doubles)
  3. local projections                          d_q = Sigma_q V_q^T (Fu_q - u_q)
  4. all-gather of d (N*k*S doubles); every rank runs the k-dimensional
     sequential sweep e_q = C_q e_{q-1} + d_q redundantly (cheaper than N-1
     serialised hops)
  5. local reconstruction + update norms        u_{q+1} = Fu_{q+1} + U_q e_q
  6. halo: the left neighbour's last u block    -> u_{q0}          (P2P)

So NCCL carries only interval-boundary states and the k-dimensional sweep
data.  Arrays hold nq+1 "blocks" of S vectors (op layout): block i is
boundary q0+i; block 0 is the halo (u0 on rank 0).

The compute of every stage is delegated to a backend (the CUDA library on
GPUs, `LibprBackend`); this module only moves data and calls collectives, so
its exchange schedule is testable on CPU with gloo and a test backend
(tests/test_parallel.py).
"""
from __future__ import annotations

import torch


def shard(total: int, rank: int, world: int):
    """Contiguous block partition: (start, count) of rank."""
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


class Comm:
    """torch.distributed wrapper (world == 1 needs no process group)."""

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

    def all_gather_cat(self, t):
        """Concatenate every rank's t (equal shapes) along dim 0, in rank order."""
        if self.world == 1:
            return t
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.cat(parts, dim=0)


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

    def nblocks(self, t) -> int:
        return (t.shape[1] if self.dim == 1 else t.shape[0]) // self.S


def parareal_sharded(backend, blocks: Blocks, u0, K: int, comm: Comm):
    """Run K Parareal iterations on this rank's intervals.

    backend: stage implementation (see LibprBackend) for intervals
             [backend.q0, backend.q0 + backend.nq) of backend.N.
    u0:      one block (S vectors) -- used by rank 0 only.
    Returns (u, upd): u holds blocks q0 .. q0+nq (block 0 = halo u_{q0});
    upd (K, N, S) = ||u^k_{q+1} - u^{k-1}_{q+1}|| for every interval q.
    """
    nq, N, S, k = backend.nq, backend.N, backend.S, backend.k
    q0 = backend.q0
    u, Fu, b = blocks.new(nq + 1), blocks.new(nq + 1), blocks.new(nq)
    backend.offsets(b)                                   # b_q = F_q 0, local q
    blocks.view(Fu, 1, nq + 1).copy_(b)                  # initialisation: Fu_{q+1} := b_q
    # reduced sweep matrices of all intervals (one P2P of U_{q0-1} + one all-gather)
    U_prev = comm.shift_right(backend.last_U())
    C_all = comm.all_gather_cat(backend.local_C(U_prev))

    def halo(arr):
        """Block 0 of arr := the left neighbour's last block (rank 0: u0)."""
        got = comm.shift_right(blocks.view(arr, nq, nq + 1).contiguous())
        blocks.view(arr, 0, 1).copy_(u0 if comm.rank == 0 else got)

    d = backend.new_d(nq)
    e_all = backend.new_d(N)
    halo(Fu)                                             # Fu_{q0} = b_{q0-1} (u0 on rank 0)
    backend.project(None, blocks.view(Fu, 0, nq), d)     # p = 0 at initialisation
    backend.sweep(C_all, comm.all_gather_cat(d), e_all)
    backend.expand(blocks.view(Fu, 1, nq + 1), e_all[q0:q0 + nq], blocks.view(u, 1, nq + 1), None)
    halo(u)
    upd = []
    for _ in range(K):
        backend.fine(blocks.view(u, 0, nq), blocks.view(Fu, 1, nq + 1), b)
        halo(Fu)
        backend.project(blocks.view(u, 0, nq), blocks.view(Fu, 0, nq), d)
        backend.sweep(C_all, comm.all_gather_cat(d), e_all)
        un = backend.new_norms(nq)
        backend.expand(blocks.view(Fu, 1, nq + 1), e_all[q0:q0 + nq], blocks.view(u, 1, nq + 1), un)
        halo(u)
        upd.append(comm.all_gather_cat(un))
    upd = torch.stack(upd).reshape(K, N, S) if K > 0 else torch.zeros((0, N, S))
    return u, upd


class LibprBackend:
    """Stages on the CUDA library (include/pr.h distributed building blocks)."""

    def __init__(self, op, G, cfg_N: int, q0: int, nq: int, m: int, k: int, S: int, source):
        self.op, self.G, self.N, self.q0, self.nq = op, G, cfg_N, q0, nq
        self.m, self.k, self.S, self.source = m, k, S, source
        self.dev = torch.device("cuda", torch.cuda.current_device())

    def new_d(self, nint: int):
        return torch.empty((nint, self.k, self.S), dtype=torch.float64, device=self.dev)

    def new_norms(self, nint: int):
        return torch.empty((nint, self.S), dtype=torch.float64, device=self.dev)

    def _ld(self, t):
        return int(t.stride(0))

    def offsets(self, out):
        from ._lib import PR_AFFINE
        self.op.fine_propagate(PR_AFFINE, self.q0, self.m, None, out, vecs_per_interval=self.S,
                               source=self.source, B=self.nq * self.S)

    def fine(self, u_in, out, b):
        from ._lib import PR_LINEAR
        self.op.fine_propagate(PR_LINEAR, self.q0, self.m, u_in, out, vecs_per_interval=self.S,
                               offset=b, B=self.nq * self.S)

    def last_U(self):
        t = torch.empty((self.op.rows, self.k), dtype=torch.float64, device=self.dev)
        self.G.export_interval(self.nq - 1, U_q=t)
        return t

    def local_C(self, U_prev):
        if U_prev is not None:
            self.G.sweep_matrices(U_prev)
        C = torch.empty((self.nq, self.k, self.k), dtype=torch.float64, device=self.dev)
        self.G.export(C=C)
        return C

    def project(self, Y1, Y2, d):
        self.G.project(self.S, Y1, Y2, self._ld(Y2), d)

    def sweep(self, C_all, d_all, e_all):
        from .api import reduced_sweep
        reduced_sweep(C_all, d_all, self.N, self.k, self.S, e_all)

    def expand(self, Fu, e_loc, out, upd):
        self.G.expand(self.S, Fu, e_loc, out, self._ld(out), upd)
