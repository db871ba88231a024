"""Dev aid: one K1P launch of a 1D config (for ncu captures): warm-up launch,
then the launch to profile.  python tools/k1p_once.py C4 16384"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_util import gpu_op  # noqa: E402
from paper_2508_08873_b200 import PR_LINEAR  # noqa: E402
from workloads.configs import get  # noqa: E402

cfg = get(sys.argv[1] if len(sys.argv) > 1 else "C4")
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.N * max(cfg.nsrc, 1)
op = gpu_op(cfg)
X = torch.randn(cfg.n, B, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for _ in range(2):
    op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y)
torch.cuda.synchronize()
print("done", flush=True)
