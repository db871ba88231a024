"""ctypes binding of libpr.so (include/pr.h).  Argument marshalling only.

Every function here forwards to the C ABI; no numerical work happens in
Python.  If the CUDA library is missing the import fails loudly -- there is
no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libpr.so")

PR_OK, PR_EINVAL, PR_EDIM, PR_ESINGULAR, PR_ENOCONV, PR_EUNAVAIL, PR_EOOM, PR_ECUDA, PR_ENCCL = range(9)
STATUS_NAMES = ["PR_OK", "PR_EINVAL", "PR_EDIM", "PR_ESINGULAR", "PR_ENOCONV", "PR_EUNAVAIL",
                "PR_EOOM", "PR_ECUDA", "PR_ENCCL"]
PR_LINEAR, PR_ADJOINT, PR_AFFINE = 0, 1, 2
PR_SRC_NONE, PR_SRC_SEP1D, PR_SRC_BUMP2D = 0, 1, 2
PR_TO_WEIGHTED, PR_FROM_WEIGHTED = 0, 1

# every symbol include/pr.h declares
EXPORTS = ["pr_last_error", "pr_version", "pr_reload_env", "pr_profile", "pr_counters", "pr_phase_counters", "pr_op_create_tridiag", "pr_op_create_pencil", "pr_op_create_weighted",
           "pr_op_weight_apply", "pr_op_create_sep2d",
           "pr_op_destroy", "pr_op_info", "pr_fine_propagate", "pr_gaussian_sketch",
           "pr_build_coarse", "pr_coarse_estimate", "pr_build_coarse_adaptive", "pr_coarse_info", "pr_coarse_factors", "pr_coarse_apply",
           "pr_coarse_destroy", "pr_parareal", "pr_parareal_tol", "pr_bounds", "pr_sequential",
           "pr_trajectory_error", "pr_efficiency", "pr_parareal_classical", "pr_coarse_sweep_matrices",
           "pr_coarse_export", "pr_coarse_export_interval", "pr_coarse_project", "pr_reduced_sweep", "pr_coarse_expand",
           "pr_comm_nccl_unique_id", "pr_comm_create_nccl", "pr_comm_create_local", "pr_comm_info",
           "pr_comm_destroy"]


class PrError(RuntimeError):
    def __init__(self, status: int, func: str, msg: str):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{func}: {name}: {msg}")
        self.status = status
        self.name = name


class Source(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("nterms", ctypes.c_int), ("nsrc", ctypes.c_int),
                ("nsteps", ctypes.c_int),
                ("space", ctypes.c_void_p), ("time", ctypes.c_void_p), ("amp", ctypes.c_void_p),
                ("gx", ctypes.c_void_p), ("gy", ctypes.c_void_p)]


class RsvdOpts(ctypes.Structure):
    _fields_ = [("power_iterations", ctypes.c_int), ("independent_adjoint", ctypes.c_int)]


_lib = None


def lib():
    """Load libpr.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise OSError(f"libpr.so not found at {SO_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(SO_PATH)
        vp, dp, ip, lg = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), ctypes.c_long
        I, D, U64 = ctypes.c_int, ctypes.c_double, ctypes.c_uint64
        sig = {
            "pr_last_error": ([], ctypes.c_char_p),
            "pr_version": ([], I),
            "pr_reload_env": ([], I),
            "pr_profile": ([I], I),
            "pr_counters": ([I, ctypes.POINTER(lg), ctypes.POINTER(lg), dp, dp, dp], I),
            "pr_phase_counters": ([I, ctypes.POINTER(lg), dp, dp], I),
            "pr_op_create_tridiag": ([I, dp, dp, dp, dp, dp, D, ctypes.POINTER(vp)], I),
            "pr_op_create_pencil": ([I, I, dp, dp, dp, dp, dp, dp, dp, D, ctypes.POINTER(vp)], I),
            "pr_op_create_weighted": ([vp, ctypes.POINTER(vp)], I),
            "pr_op_weight_apply": ([vp, I, I, vp, lg, vp, lg, vp], I),
            "pr_op_create_sep2d": ([I, D, ctypes.POINTER(vp)], I),
            "pr_op_destroy": ([vp], I),
            "pr_op_info": ([vp, ctypes.POINTER(lg), ip, ip], I),
            "pr_fine_propagate": ([vp, I, I, I, I, I, ctypes.POINTER(Source), vp, lg, vp, lg, vp, lg, vp], I),
            "pr_gaussian_sketch": ([vp, I, I, I, U64, vp, lg, vp], I),
            "pr_build_coarse": ([vp, I, I, I, I, I, I, U64, ctypes.POINTER(RsvdOpts), vp, vp, ctypes.POINTER(vp)], I),
            "pr_coarse_estimate": ([vp, vp, I, U64, dp, vp], I),
            "pr_build_coarse_adaptive": ([vp, I, I, I, I, I, I, I, D, I, U64, ctypes.POINTER(RsvdOpts), vp, vp,
                                          ctypes.POINTER(vp), ip], I),
            "pr_coarse_info": ([vp, ip, ip, ip, ip, ip, dp, dp, dp, ip], I),
            "pr_coarse_factors": ([vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)], I),
            "pr_coarse_apply": ([vp, I, I, vp, lg, vp, lg, vp], I),
            "pr_coarse_destroy": ([vp], I),
            "pr_parareal": ([vp, vp, I, vp, lg, ctypes.POINTER(Source), I, vp, lg, dp, dp, vp, lg, vp], I),
            "pr_parareal_tol": ([vp, vp, I, vp, lg, ctypes.POINTER(Source), I, D, vp, lg, dp, dp, vp, lg, ip, vp], I),
            "pr_bounds": ([D, D, I, I, dp, dp, dp, dp, dp], I),
            "pr_sequential": ([vp, I, vp, lg, ctypes.POINTER(Source), I, I, vp, lg, vp], I),
            "pr_trajectory_error": ([vp, I, I, I, vp, lg, vp, lg, dp, dp, vp], I),
            "pr_efficiency": ([D, D, I, I, dp, dp, dp], I),
            "pr_parareal_classical": ([vp, ctypes.POINTER(Source), vp, I, vp, lg, ctypes.POINTER(Source), I, I, I,
                                       vp, lg, dp, vp, lg, vp], I),
            "pr_coarse_sweep_matrices": ([vp, vp, vp], I),
            "pr_coarse_export": ([vp, vp, vp, vp, vp, vp], I),
            "pr_coarse_export_interval": ([vp, I, vp, vp, vp], I),
            "pr_coarse_project": ([vp, I, vp, vp, lg, vp, vp], I),
            "pr_reduced_sweep": ([vp, vp, I, I, I, vp, vp], I),
            "pr_coarse_expand": ([vp, I, vp, vp, vp, lg, vp, vp], I),
            "pr_comm_nccl_unique_id": ([vp], I),
            "pr_comm_create_nccl": ([I, I, vp, ctypes.POINTER(vp)], I),
            "pr_comm_create_local": ([I, ctypes.POINTER(vp)], I),
            "pr_comm_info": ([vp, ip, ip], I),
            "pr_comm_destroy": ([vp], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def check(status: int, func: str):
    if status != PR_OK:
        msg = lib().pr_last_error()
        raise PrError(status, func, msg.decode() if msg else "")
    return status
