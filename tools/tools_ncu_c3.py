"""One C3 build (for ncu on the K2 DMMA GEMM)."""
import torch
from paper_2508_08873_b200 import Operator, Coarse
from workloads.configs import get
cfg = get("C3")
op = Operator.sep2d(cfg.n, cfg.dt)
G = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
print(G.info()["delta"])
