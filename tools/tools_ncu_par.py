"""One C4 Parareal run (for ncu on the affine stepper / sweep / expand)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_08873_b200 import Operator, Coarse, SourceTerm, parareal
from workloads import generators as G
from workloads.configs import get
import dataclasses, sys
cfg = get("C4")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rs, cs = G.operator_1d_sums(cfg)
op = Operator.tridiag(*G.operator_1d(cfg), cfg.dt, rowsum=rs, colsum=cs)
Gc = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
S = cfg.nsrc
u0 = torch.tensor(np.ascontiguousarray(np.stack([G.initial_value(cfg)] * S).T), dtype=torch.float64, device="cuda")
U = torch.empty((cfg.n, (cfg.N + 1) * S), dtype=torch.float64, device="cuda")
src = SourceTerm.sep1d(*G.source_1d(cfg))
upd, bn = parareal(Gc, op, u0, src, K, U, nsrc=S)
torch.cuda.synchronize()
print("done", upd[-1, -1, :3])
