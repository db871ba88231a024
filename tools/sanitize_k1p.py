"""Dev aid for compute-sanitizer: small K1P launches (LINEAR, ADJOINT, AFFINE)
on a C2-shaped and a C4-shaped operator, plus a pencil (Exp 2) fine solve."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from dataclasses import replace  # noqa: E402

from gpu_util import gpu_op, gpu_source  # noqa: E402
from paper_2508_08873_b200 import PR_ADJOINT, PR_AFFINE, PR_LINEAR  # noqa: E402
from workloads.configs import get  # noqa: E402

for name, B in (("C2", 48), ("T4", 40), ("E2", 20)):
    cfg = get(name)
    if name == "C2":
        cfg = replace(cfg, m=6)
    op = gpu_op(cfg)
    X = torch.randn(cfg.n, B, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    for mode in (PR_LINEAR, PR_ADJOINT):
        op.fine_propagate(mode, 0, cfg.m, X, Y)
    S = cfg.nsrc
    op.fine_propagate(PR_AFFINE, 0, cfg.m, None, Y, vecs_per_interval=S, source=gpu_source(cfg), B=(B // S) * S)
    torch.cuda.synchronize()
    print(name, "ok", flush=True)
