"""Dev aid: CholeskyQR pass counts (Y, Z) of a C4 build and the build's kernel times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from gpu_util import gpu_op
from paper_2508_08873_b200 import Coarse
from workloads.configs import get
cfg = get(sys.argv[1] if len(sys.argv) > 1 else "C4")
op = gpu_op(cfg)
for it in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    G = Coarse.build(op, cfg.N, cfg.m, cfg.k, cfg.p, cfg.seed_omega)
    b.record()
    torch.cuda.synchronize()
    info = G.info()
    print({k: v for k, v in info.items() if k != "sigma"}, f"build {a.elapsed_time(b):.1f} ms")
    G.close()
