"""Dev aid: per-phase clock64 breakdown of the partitioned stepper (PR_PART_PROF)."""
import os
import sys

import torch

os.environ["PR_PART_PROF"] = "1"
os.environ["PR_FORCE_PART"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "tests"))
from gpu_util import gpu_op  # noqa: E402
from paper_2508_08873_b200 import PR_LINEAR, build  # noqa: E402
from workloads.configs import get  # noqa: E402

build.build()
for name in sys.argv[1:] or ["C2", "C1"]:
    cfg = get(name)
    op = gpu_op(cfg)
    X = torch.randn(cfg.n, int(os.environ.get("PB", "64")), dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y)
    torch.cuda.synchronize()
