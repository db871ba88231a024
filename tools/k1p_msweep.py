"""Dev aid: K1P launch time against the number of steps m (C4 operator, B vectors):
the intercept is the per-group prologue/epilogue cost, the slope the cost of a step.
    python tools/k1p_msweep.py [B]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_util import gpu_op  # noqa: E402
from paper_2508_08873_b200 import PR_LINEAR  # noqa: E402
from workloads.configs import get  # noqa: E402

cfg = get("C4")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
op = gpu_op(cfg)
X = torch.randn(cfg.n, B, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for m in (1, 2, 16, 32, 64, 128):
    for _ in range(2):
        op.fine_propagate(PR_LINEAR, 0, m, X, Y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        op.fine_propagate(PR_LINEAR, 0, m, X, Y)
    b.record()
    torch.cuda.synchronize()
    print(f"m={m:4d}: {a.elapsed_time(b) / 3:.3f} ms/launch", flush=True)
