"""One C3 build (for ncu on the K2 DMMA GEMM)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from paper_2508_08873_b200 import Operator, Coarse
from workloads.configs import get
cfg = get("C3")
op = Operator.sep2d(cfg.n, cfg.dt)
G = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
print(G.info()["delta"])
