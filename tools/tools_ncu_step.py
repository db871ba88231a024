"""One stepper launch at C4 build size (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import sys
import torch
from paper_2508_08873_b200 import Operator, PR_LINEAR
from workloads import generators as G
from workloads.configs import get
cfg = get(sys.argv[1] if len(sys.argv) > 1 else "C4")
rs, cs = G.operator_1d_sums(cfg)
op = Operator.tridiag(*G.operator_1d(cfg), cfg.dt, rowsum=rs, colsum=cs)
B = cfg.N * cfg.l
m = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.m
X = torch.randn((cfg.n, B), dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
op.fine_propagate(PR_LINEAR, 0, m, X, Y, vecs_per_interval=cfg.l)
torch.cuda.synchronize()
print("done")
