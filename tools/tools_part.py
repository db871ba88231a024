"""Dev aid: time the fused (K1) and partitioned (K1P) 1D steppers on C2/C1-shaped
fine solves over a range of batch sizes (CUDA events, after warm-up)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "tests"))
from gpu_util import gpu_op  # noqa: E402
from paper_2508_08873_b200 import PR_LINEAR, build  # noqa: E402
from workloads.configs import get  # noqa: E402

build.build()
for name in sys.argv[1:] or ["C2", "C1"]:
    cfg = get(name)
    op = gpu_op(cfg)
    for B in [int(b) for b in os.environ.get("BLIST", "32,64,128,256,512,1024,2560").split(",")]:
        X = torch.randn(cfg.n, B, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(X)
        res = {}
        for path in ("fused", "part"):
            os.environ.pop("PR_NO_PART", None)
            os.environ.pop("PR_FORCE_PART", None)
            os.environ["PR_NO_PART" if path == "fused" else "PR_FORCE_PART"] = "1"
            for _ in range(2):
                op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            a.record()
            for _ in range(reps):
                op.fine_propagate(PR_LINEAR, 0, cfg.m, X, Y)
            b.record()
            torch.cuda.synchronize()
            res[path] = a.elapsed_time(b) / reps
            res[path + "_y"] = Y.clone()
        err = (res["fused_y"] - res["part_y"]).abs().max().item() / res["fused_y"].abs().max().item()
        print(f"{name} n={cfg.n} m={cfg.m} B={B}: fused {res['fused']:.3f} ms  part {res['part']:.3f} ms  "
              f"relmax {err:.2e}", flush=True)
