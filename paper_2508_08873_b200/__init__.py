"""B200-native hot path of the spectral-coarse-solver Parareal (arXiv 2508.08873).

The compute runs in libpr.so (hand-written sm_100a CUDA, C ABI in
include/pr.h); this package is its ctypes binding.  There is no CPU
fallback: the first call raises OSError if libpr.so has not been built
(`python -c "import __graft_entry__ as g; g.build()"`).
"""
from .api import (Coarse, Comm, Operator, SourceTerm, bounds, counters, efficiency, parareal,  # noqa: F401
                  parareal_classical, parareal_tol, profile, sequential, trajectory_error)
from ._lib import PR_ADJOINT, PR_AFFINE, PR_LINEAR, PrError, lib  # noqa: F401


def require_cuda():
    """Load libpr.so and check a CUDA device is present (raises otherwise)."""
    import torch
    lib()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2508_08873_b200 needs a CUDA device (B200, sm_100a)")
