"""Run the oracle's per-interval rSVD (oracle/rsvd.py, as it stands) for many
intervals in parallel worker processes -- test harness only.  The intervals
are independent; each worker is single-threaded (OpenMP / BLAS
pinned to one thread) so the pool uses every host core once."""
from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor
import multiprocessing as mp


def _init():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def _one(args):
    cfg, n = args
    from oracle.fine import make_op
    from oracle.rsvd import rsvd_interval
    return rsvd_interval(make_op(cfg), n, cfg.k, cfg.p, cfg.seed_omega)


def rsvd_intervals(cfg, intervals=None, workers=None):
    """[rsvd_interval(op, n, ...) for n in intervals] (1-based, default 1..N)."""
    intervals = list(range(1, cfg.N + 1)) if intervals is None else list(intervals)
    workers = workers or max(1, min(len(intervals), os.cpu_count() or 1))
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"), initializer=_init) as ex:
        return list(ex.map(_one, [(cfg, n) for n in intervals]))
