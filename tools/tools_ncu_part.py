"""Dev aid: one forced-partitioned C2 fine solve (B=64) for an ncu capture."""
import os
import sys

import torch

os.environ["PR_FORCE_PART"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "tests"))
from gpu_util import gpu_op  # noqa: E402
from paper_2508_08873_b200 import PR_LINEAR, build  # noqa: E402
from workloads.configs import get  # noqa: E402

build.build()
cfg = get(sys.argv[1] if len(sys.argv) > 1 else "C2")
op = gpu_op(cfg)
X = torch.randn(cfg.n, 64, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for _ in range(2):
    op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y)
torch.cuda.synchronize()
print("ok")
