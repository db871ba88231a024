"""Multi-GPU bootstrap of the interval-sharded path (one process per GPU).

The sharded rSVD build and Parareal schedule live in libpr behind the C ABI
(include/pr.h "distribution"): `Coarse.build(...,
comm=c)` builds rank r's block of intervals, `parareal(G, ...)` runs the
collective schedule, and the library moves the interval-boundary data itself
(NCCL send/recv of one boundary block per half-iteration, all-gather of the
k-dimensional sweep data, max-reduction of delta and eps).  This module only
creates the communicator from an existing torch.distributed process group:
rank 0 makes the NCCL unique id, the group broadcasts it, every rank joins.
"""
from __future__ import annotations

import torch


def shard(total: int, rank: int, world: int):
    """Contiguous block partition (start, count) of `total` intervals -- the
    partition libpr uses for a communicator of `world` ranks."""
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def broadcast_bytes(payload: bytes, nbytes: int, group=None, device=None) -> bytes:
    """Rank 0's `payload` (nbytes long) on every rank of the process group."""
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().tolist())


def nccl_comm(group=None, api=None):
    """pr_comm over the ranks of a torch.distributed group (one GPU each, the
    current device).  `api` defaults to paper_2508_08873_b200.Comm (tests
    substitute a host-only stand-in)."""
    import torch.distributed as dist
    if api is None:
        from .api import Comm as api
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = api.nccl_unique_id() if rank == 0 else bytes(128)
    dev = None
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    uid = broadcast_bytes(uid, 128, group, dev)
    return api.nccl(rank, world, uid)
