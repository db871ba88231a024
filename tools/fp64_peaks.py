"""Measure the FP64 roofline denominators on this GPU and write
profiles/fp64_peaks.json (bench.py reads it):
  dfma_tflops         FP64 FMA pipe, all SMs (tools/ub/fp64_peaks.cu)
  dmma_m8n8k4_tflops  FP64 tensor pipe (mma.sync m8n8k4, the DMMA the 2D path uses)
  dgemm_tflops        cuBLAS DGEMM 8192^3 through torch.matmul (best of 5)
"""
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ub = os.path.join(ROOT, "tools", "ub")
exe = os.path.join(ub, "fp64_peaks")
if not os.path.exists(exe):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-o", exe, exe + ".cu"])
res = json.loads(subprocess.check_output([exe]).decode().strip().splitlines()[-1])
n = 8192
a = torch.randn((n, n), dtype=torch.float64, device="cuda")
b = torch.randn((n, n), dtype=torch.float64, device="cuda")
torch.matmul(a, b)
best = 0.0
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
res["dgemm_tflops"] = round(best, 3)
res["gpu"] = torch.cuda.get_device_name()
res["how"] = "tools/fp64_peaks.py: DFMA / DMMA microkernels (best of 5, CUDA events) and torch.matmul fp64 8192^3"
out = os.path.join(ROOT, "profiles", sys.argv[1] if len(sys.argv) > 1 else "fp64_peaks.json")
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
