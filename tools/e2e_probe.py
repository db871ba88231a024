"""Dev aid: where the end-to-end step (bench.py _e2e) spends its host-visible time.
Each phase is bracketed by torch.cuda.synchronize() and timed on the host."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_08873_b200 import Coarse, Operator, SourceTerm, parareal  # noqa: E402
from workloads.configs import get  # noqa: E402

cfg = get(sys.argv[1] if len(sys.argv) > 1 else "C4")
dev = torch.device("cuda", 0)
wl = bench.Workload(cfg, 0, 1, dev)
c = cfg
pin = {k: torch.from_numpy(np.ascontiguousarray(wl.host[k])).pin_memory() for k in ("space", "time", "amp", "u0")}
out_host = torch.empty(tuple(wl.U.shape), dtype=torch.float64).pin_memory()


def tick(label, t0):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"  {label:28s} {1e3 * (t1 - t0):9.2f} ms", flush=True)
    return t1


for it in range(3):
    print(f"step {it}")
    torch.cuda.synchronize()
    t = time.perf_counter()
    dv = {k: v.to(dev, non_blocking=True) for k, v in pin.items()}
    t = tick("h2d", t)
    rs, cs = wl.host["sums"]
    op = Operator.tridiag(*wl.host["op"], c.dt, rowsum=rs, colsum=cs)
    t = tick("Operator.tridiag", t)
    src = SourceTerm(1, dv["time"].shape[0], dv["amp"].shape[0], dv["time"].shape[1],
                     {"space": dv["space"], "time": dv["time"], "amp": dv["amp"]})
    t = tick("SourceTerm", t)
    G = Coarse.build(op, c.N, c.m, c.k, c.p, c.seed_omega)
    t = tick("Coarse.build", t)
    upd, bn = parareal(G, op, dv["u0"], src, c.K, wl.U, nsrc=wl.ns)
    t = tick("parareal", t)
    out_host.copy_(wl.U, non_blocking=True)
    t = tick("d2h", t)
    G.close() if hasattr(G, "close") else None
    t = tick("G.close", t)
    op.close()
    t = tick("op.close", t)
