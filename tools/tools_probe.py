"""Quick timing probe of the 1D stepper (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import sys, time
import numpy as np
import torch
from paper_2508_08873_b200 import Operator, PR_LINEAR, Coarse
from workloads import generators as G
from workloads.configs import get

for name in sys.argv[1:] or ["C4"]:
    cfg = get(name)
    rs, cs = G.operator_1d_sums(cfg)
    op = Operator.tridiag(*G.operator_1d(cfg), cfg.dt, rowsum=rs, colsum=cs)
    B = cfg.N * cfg.l
    X = torch.randn((cfg.n, B), dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    for _ in range(2):
        op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y, vecs_per_interval=cfg.l)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    R = 5
    for _ in range(R):
        op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y, vecs_per_interval=cfg.l)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    dofsteps = cfg.n * B * cfg.m
    print(f"{name}: stepper B={B} n={cfg.n} m={cfg.m}: {ms:.3f} ms  {dofsteps/ms/1e-3:.3e} DOF-steps/s  "
          f"{16*dofsteps/ms/1e6:.1f} GB/s @16B/DOF-step", flush=True)
    t0 = time.time()
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gc.info()
    torch.cuda.synchronize()
    t1 = time.time()
    Gc.close()
    Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    info = Gc.info()
    t2 = time.time()
    print(f"{name}: build {1e3*(t1-t0):.1f} ms (first) {1e3*(t2-t1):.1f} ms; qr passes {info['qr_passes']} delta {info['delta']:.6f} eps {info['eps']:.3e}", flush=True)
