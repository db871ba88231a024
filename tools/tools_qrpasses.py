import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import sys, time, torch
from paper_2508_08873_b200 import Operator, Coarse
from workloads import generators as G
from workloads.configs import get
for name in sys.argv[1:]:
    cfg = get(name)
    if cfg.dim == 1:
        rs, cs = G.operator_1d_sums(cfg)
        op = Operator.tridiag(*G.operator_1d(cfg), cfg.dt, rowsum=rs, colsum=cs)
    else:
        op = Operator.sep2d(cfg.n, cfg.dt)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.time()
        Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
        info = Gc.info()
        t1 = time.time()
        print(name, "build %.1f ms" % (1e3 * (t1 - t0)), "qr_passes (enqueued)", info["qr_passes"], flush=True)
        Gc.close()
