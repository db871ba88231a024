import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import os, sys
import numpy as np
import torch
from paper_2508_08873_b200 import Operator, Coarse
from workloads import generators as G
from workloads.configs import get
cfg = get(sys.argv[1] if len(sys.argv) > 1 else "C1")
rs, cs = G.operator_1d_sums(cfg)
op = Operator.tridiag(*G.operator_1d(cfg), cfg.dt, rowsum=rs, colsum=cs)
print("op ok", flush=True)
Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
print("build queued", flush=True)
info = Gc.info(raise_on_error=False)
print(info["qr_passes"], info["status"], info["sigma"][0][:4], flush=True)
