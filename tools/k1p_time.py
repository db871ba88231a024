"""Dev aid: device time of one 1D fine-propagation launch (K1P unless
PR_NO_PART=1) per config / batch / mode, CUDA events, after warm-up.
    python tools/k1p_time.py C4 16384 [linear|adjoint|affine|offset] [reps]
(offset: LINEAR with a stored offset added, as in a Parareal iteration)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_util import gpu_op, gpu_source  # noqa: E402
from paper_2508_08873_b200 import PR_ADJOINT, PR_AFFINE, PR_LINEAR  # noqa: E402
from workloads.configs import get  # noqa: E402

cfg = get(sys.argv[1] if len(sys.argv) > 1 else "C4")
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.N * max(cfg.nsrc, 1)
mode = sys.argv[3] if len(sys.argv) > 3 else "linear"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
op = gpu_op(cfg)
X = torch.randn(cfg.n, B, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
src = gpu_source(cfg) if mode == "affine" else None
OFF = torch.randn_like(X) if mode == "offset" else None
S = cfg.nsrc if mode == "affine" else 1


def run():
    if mode == "affine":
        op.fine_propagate(PR_AFFINE, 0, cfg.m, None, Y, vecs_per_interval=S, source=src)
    else:
        op.fine_propagate(PR_ADJOINT if mode == "adjoint" else PR_LINEAR, 0, cfg.m, X, Y, offset=OFF)


for _ in range(3):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
dof = cfg.n * B * cfg.m
print(f"{cfg.name} n={cfg.n} m={cfg.m} B={B} {mode}: {ms:.3f} ms/launch  {dof / ms / 1e9:.3f} GDOF-steps/s "
      f"({5 * dof / ms / 1e9:.2f} TF/s at 5 flop/DOF-step)", flush=True)
