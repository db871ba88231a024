"""Dev aid: C2 partitioned stepper at L=32 (default) vs L=64 (PR_PART_L=64), B=64."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, "tests")
from gpu_util import gpu_op
from paper_2508_08873_b200 import PR_LINEAR
from workloads.configs import get
os.environ["PR_FORCE_PART"] = "1"
cfg = get(sys.argv[1])
op = gpu_op(cfg)
for B in (32, 64, 256):
    X = torch.randn(cfg.n, B, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
    for _ in range(2): op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y)
    b.record(); torch.cuda.synchronize()
    print(os.environ.get("PR_PART_L", "32"), cfg.name, "B", B, round(a.elapsed_time(b) / 5, 4), "ms", flush=True)
'''
for L in ("32", "64"):
    env = dict(os.environ)
    if L == "64":
        env["PR_PART_L"] = "64"
    subprocess.run([sys.executable, "-c", code, sys.argv[1] if len(sys.argv) > 1 else "C2"], env=env)
