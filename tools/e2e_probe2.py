"""Dev aid: the end-to-end step of bench.py (_e2e, serial copy) without host synchronisation
between its phases: CUDA events on the compute stream give the device timeline, host clocks
the time the host spends in each call."""
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda", 0)
wl = bench.Workload(cfg, 0, 1, dev)
c = cfg
for _ in range(2):
    wl.step()
torch.cuda.synchronize()
pin = {k: torch.from_numpy(np.ascontiguousarray(wl.host[k])).pin_memory() for k in ("space", "time", "amp", "u0")}
out_host = torch.empty(tuple(wl.U.shape), dtype=torch.float64).pin_memory()
names = ["h2d", "op create", "build", "parareal", "d2h", "close"]
ev, host = [], []


def mark():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    ev[-1].append(e)
    host[-1].append(time.perf_counter())


torch.cuda.synchronize()
for it in range(steps):
    ev.append([])
    host.append([])
    mark()
    dv = {k: v.to(dev, non_blocking=True) for k, v in pin.items()}
    mark()
    rs, cs = wl.host["sums"]
    op = Operator.tridiag(*wl.host["op"], c.dt, rowsum=rs, colsum=cs)
    src = SourceTerm(1, dv["time"].shape[0], dv["amp"].shape[0], dv["time"].shape[1],
                     {"space": dv["space"], "time": dv["time"], "amp": dv["amp"]})
    mark()
    G = Coarse.build(op, c.N, c.m, c.k, c.p, c.seed_omega)
    mark()
    upd, bn = parareal(G, op, dv["u0"], src, c.K, wl.U, nsrc=wl.ns)
    mark()
    out_host.copy_(wl.U, non_blocking=True)
    mark()
    G.close()
    op.close()
    mark()
torch.cuda.synchronize()
for it in range(steps):
    dts = [ev[it][i].elapsed_time(ev[it][i + 1]) for i in range(6)]
    hts = [1e3 * (host[it][i + 1] - host[it][i]) for i in range(6)]
    print(f"step {it}: device " + "  ".join(f"{n} {d:.1f}" for n, d in zip(names, dts)) + f"  | total {sum(dts):.1f} ms")
    print(f"        host   " + "  ".join(f"{n} {d:.1f}" for n, d in zip(names, hts)) + f"  | total {sum(hts):.1f} ms")
print(f"all steps, first event to last: {ev[0][0].elapsed_time(ev[-1][-1]) / steps:.1f} ms per step")
