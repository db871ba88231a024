"""Build libpr.so (the CUDA path) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libpr.so")
STAMP = SO + ".stamp"
SRC = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HDR = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
    os.path.join(os.path.dirname(HERE), "include", "pr.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "550"]


def _fingerprint(extra) -> str:
    """Content hash of every source and header plus the exact compiler flags:
    a library built from other sources or flags (e.g. a PR_EXTRA_NVCC_FLAGS
    probe build) is never reused."""
    h = hashlib.sha256()
    for f in SRC + HDR:
        h.update(f.encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(NVCC_FLAGS + list(extra)).encode())
    return h.hexdigest()


def _stale(fp: str) -> bool:
    if not os.path.exists(SO) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != fp


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu to an object in parallel (one nvcc per file), then link
    the shared library.  PR_EXTRA_NVCC_FLAGS adds flags (e.g. -DPR_PART_PROBES)."""
    extra = os.environ.get("PR_EXTRA_NVCC_FLAGS", "").split()
    fp = _fingerprint(extra)
    if force or _stale(fp):
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        cflags = [f for f in NVCC_FLAGS if f != "-shared"] + extra
        objdir = os.path.join(HERE, "build_obj")
        os.makedirs(objdir, exist_ok=True)
        objs, procs = [], []
        for src in SRC:
            obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
            cmd = [nvcc] + cflags + ["-c", "-o", obj, src]
            if verbose:
                print(" ".join(cmd))
            procs.append((subprocess.Popen(cmd, cwd=os.path.join(HERE, "csrc")), cmd))
            objs.append(obj)
        failed = [cmd for p, cmd in procs if p.wait() != 0]
        if failed:
            raise subprocess.CalledProcessError(1, failed[0])
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
               "-o", SO + ".tmp"] + objs + ["-ldl"]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(SO + ".tmp", SO)
        with open(STAMP, "w") as f:
            f.write(fp + "\n")
    return SO


if __name__ == "__main__":
    print(build(force=True, verbose=True))
