import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import sys, torch
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
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gc.info()
    U = torch.empty((op.rows, cfg.k), dtype=torch.float64, device="cuda")
    V = torch.empty_like(U)
    worst = 0.0
    for q in range(cfg.N):
        Gc.export_interval(q, U_q=U, V_q=V)
        I = torch.eye(cfg.k, dtype=torch.float64, device="cuda")
        e = max(float((U.T @ U - I).abs().max()), float((V.T @ V - I).abs().max()))
        worst = max(worst, e)
    print(name, "max |U^T U - I|, |V^T V - I| over intervals:", worst, "qr", info["qr_passes"], flush=True)
