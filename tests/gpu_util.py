"""Test helpers: move seeded workload inputs between the oracle's layout and
the CUDA path's op layout (pure data movement), and set up operators/sources
for the CUDA path from the same generators the oracle uses."""
from __future__ import annotations

import numpy as np

from workloads import generators as G

TAU_1D = 1e-10      # BASELINE.json north_star tolerance for fp64 states and sigmas
TAU_2D = 1e-8       # ... on the 2D GEMM paths


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def gpu_op(cfg):
    from paper_2508_08873_b200 import Operator
    if cfg.problem.startswith("exp2"):             # time-dependent pencil (workloads/exp2.py)
        from workloads import exp2
        L, rs, M = exp2.step_matrices(cfg.problem, cfg.n, cfg.T, cfg.N * cfg.m)
        return Operator.pencil(*L, cfg.dt, lrowsum=rs, mass=M)
    if cfg.dim == 1:
        rs, cs = G.operator_1d_sums(cfg)
        return Operator.tridiag(*G.operator_1d(cfg), cfg.dt, rowsum=rs, colsum=cs)
    return Operator.sep2d(cfg.n, cfg.dt)


def gpu_source(cfg):
    from paper_2508_08873_b200 import SourceTerm
    if cfg.dim == 1:
        return SourceTerm.sep1d(*G.source_1d(cfg))
    gx, gy = G.source_2d(cfg)
    return SourceTerm.bump2d(G.pad1d_last(gx), G.pad1d_last(gy))


def to_gpu(cfg, X: np.ndarray, ld: int = None):
    """Oracle batch (nvec, n) / (nvec, n, n) -> op-layout CUDA tensor."""
    import torch
    X = np.asarray(X, dtype=np.float64)
    nvec = X.shape[0]
    if cfg.dim == 1:
        ld = ld or nvec
        out = np.zeros((cfg.n, ld))
        out[:, :nvec] = X.T
    else:
        P = cfg.n + 1
        ld = ld or P * P
        out = np.zeros((nvec, ld))
        out[:, : P * P] = G.pad2d(X).reshape(nvec, P * P)
    return torch.tensor(out, dtype=torch.float64, device="cuda")


def from_gpu(cfg, T, nvec: int = None) -> np.ndarray:
    """Op-layout CUDA tensor -> oracle batch layout."""
    A = T.detach().cpu().numpy()
    if cfg.dim == 1:
        nvec = nvec or A.shape[1]
        return np.ascontiguousarray(A[:, :nvec].T)
    P = cfg.n + 1
    nvec = nvec or A.shape[0]
    return G.unpad2d(A[:nvec, : P * P].reshape(nvec, P, P))


def empty_batch(cfg, nvec: int, ld: int = None):
    import torch
    if cfg.dim == 1:
        return torch.zeros((cfg.n, ld or nvec), dtype=torch.float64, device="cuda")
    P = cfg.n + 1
    return torch.zeros((nvec, ld or P * P), dtype=torch.float64, device="cuda")


def relnorm(a, b, scale=None):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    s = scale if scale is not None else max(np.linalg.norm(b), 1e-300)
    return d / s
