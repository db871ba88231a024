"""Python API over the C ABI (include/pr.h): handles + torch-tensor marshalling.

Tensors are CUDA fp64 tensors in the operator's layout:
  1D: a batch of B vectors is a (n, ld) row-major tensor, vector c = column c;
  2D: a batch of B vectors is a (B, ld) tensor (ld >= (n+1)^2), vector c =
      row c, each a padded (n+1) x (n+1) grid with a zero ghost row/col 0.
No arithmetic of the method runs here; see include/pr.h for the semantics.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as L
from ._lib import PR_ADJOINT, PR_AFFINE, PR_LINEAR, check  # noqa: F401


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    if t is None:
        return None
    assert t.is_cuda and t.dtype == torch.float64, "expected a CUDA float64 tensor"
    return ctypes.c_void_p(t.data_ptr())


def _hptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ld(t, dim: int) -> int:
    """Leading dimension of a 1D (n, ld) or 2D (B, ld) batch tensor."""
    assert t.dim() == 2 and (t.stride(1) == 1 or t.shape[1] == 1), \
        "batch tensors must be 2D with unit inner stride"
    if t.shape[0] == 1:             # a single row: any leading stride >= its length works
        return max(int(t.stride(0)), int(t.shape[1]))
    return int(t.stride(0))


class Operator:
    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        rows = ctypes.c_long()
        dim = ctypes.c_int()
        n = ctypes.c_int()
        check(L.lib().pr_op_info(self._h, ctypes.byref(rows), ctypes.byref(dim), ctypes.byref(n)),
              "pr_op_info")
        self.rows, self.dim, self.n = rows.value, dim.value, n.value

    @classmethod
    def tridiag(cls, sub, diag, sup, dt: float, rowsum=None, colsum=None) -> "Operator":
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (sub, diag, sup)]
        rs = None if rowsum is None else np.ascontiguousarray(rowsum, dtype=np.float64)
        cs = None if colsum is None else np.ascontiguousarray(colsum, dtype=np.float64)
        h = ctypes.c_void_p()
        check(L.lib().pr_op_create_tridiag(len(arrs[1]), *[_hptr(a) for a in arrs],
                                           _hptr(rs) if rs is not None else None,
                                           _hptr(cs) if cs is not None else None,
                                           float(dt), ctypes.byref(h)), "pr_op_create_tridiag")
        return cls(h)

    @classmethod
    def pencil(cls, lsub, ldiag, lsup, dt: float, lrowsum=None, mass=None) -> "Operator":
        """Time-dependent pencil: (nsteps, n) arrays of the step matrices
        M + dt A(t_g); mass = (msub, mdiag, msup) or None (M = I)."""
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (lsub, ldiag, lsup)]
        nsteps, n = arrs[1].shape
        rs = None if lrowsum is None else np.ascontiguousarray(lrowsum, dtype=np.float64)
        ms = [None] * 3 if mass is None else [np.ascontiguousarray(a, dtype=np.float64) for a in mass]
        h = ctypes.c_void_p()
        check(L.lib().pr_op_create_pencil(int(n), int(nsteps), *[_hptr(a) for a in arrs],
                                          _hptr(rs) if rs is not None else None,
                                          *[_hptr(a) if a is not None else None for a in ms],
                                          float(dt), ctypes.byref(h)), "pr_op_create_pencil")
        return cls(h)

    def weighted(self) -> "Operator":
        """The view in the mass-matrix inner product (pr_op_create_weighted);
        keeps this operator alive."""
        h = ctypes.c_void_p()
        check(L.lib().pr_op_create_weighted(self._h, ctypes.byref(h)), "pr_op_create_weighted")
        v = Operator(h)
        v._base = self
        return v

    def to_weighted(self, X, Y, stream=None):
        check(L.lib().pr_op_weight_apply(self._h, L.PR_TO_WEIGHTED, int(X.shape[1]), _ptr(X), _ld(X, 1), _ptr(Y),
                                         _ld(Y, 1), _stream(stream)), "pr_op_weight_apply")
        return Y

    def from_weighted(self, X, Y, stream=None):
        check(L.lib().pr_op_weight_apply(self._h, L.PR_FROM_WEIGHTED, int(X.shape[1]), _ptr(X), _ld(X, 1),
                                         _ptr(Y), _ld(Y, 1), _stream(stream)), "pr_op_weight_apply")
        return Y

    @classmethod
    def sep2d(cls, n: int, dt: float) -> "Operator":
        h = ctypes.c_void_p()
        check(L.lib().pr_op_create_sep2d(int(n), float(dt), ctypes.byref(h)), "pr_op_create_sep2d")
        return cls(h)

    def close(self):
        if self._h:
            L.lib().pr_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def fine_propagate(self, mode: int, first_interval: int, m: int, U_in, U_out,
                       vecs_per_interval: int = 1, source: "SourceTerm" = None, offset=None,
                       B: int = None, stream=None):
        if B is None:
            B = U_out.shape[1] if self.dim == 1 else U_out.shape[0]
        src = ctypes.byref(source.struct) if source is not None else None
        check(L.lib().pr_fine_propagate(
            self._h, int(mode), int(first_interval), int(m), int(B), int(vecs_per_interval), src,
            _ptr(U_in), _ld(U_in, self.dim) if U_in is not None else 0,
            _ptr(U_out), _ld(U_out, self.dim),
            _ptr(offset), _ld(offset, self.dim) if offset is not None else 0,
            _stream(stream)), "pr_fine_propagate")
        return U_out

    def gaussian_sketch(self, first_interval: int, n_intervals: int, l: int, seed: int, out,
                        stream=None):
        check(L.lib().pr_gaussian_sketch(self._h, int(first_interval), int(n_intervals), int(l),
                                         ctypes.c_uint64(int(seed)), _ptr(out), _ld(out, self.dim),
                                         _stream(stream)), "pr_gaussian_sketch")
        return out


class SourceTerm:
    """Keeps the device tensors alive alongside the pr_source struct."""

    def __init__(self, kind, nterms, nsrc, nsteps, tensors: dict):
        self.tensors = tensors
        st = L.Source()
        st.kind, st.nterms, st.nsrc, st.nsteps = kind, nterms, nsrc, nsteps
        for key in ("space", "time", "amp", "gx", "gy"):
            t = tensors.get(key)
            setattr(st, key, t.data_ptr() if t is not None else None)
        self.struct = st

    @classmethod
    def sep1d(cls, space, time, amp, device="cuda") -> "SourceTerm":
        t = {k: torch.as_tensor(np.ascontiguousarray(v), dtype=torch.float64, device=device)
             for k, v in (("space", space), ("time", time), ("amp", amp))}
        R, nsteps = t["time"].shape
        return cls(L.PR_SRC_SEP1D, R, t["amp"].shape[0], nsteps, t)

    @classmethod
    def bump2d(cls, gx_padded, gy_padded, device="cuda") -> "SourceTerm":
        t = {k: torch.as_tensor(np.ascontiguousarray(v), dtype=torch.float64, device=device)
             for k, v in (("gx", gx_padded), ("gy", gy_padded))}
        nb, nsteps, _ = t["gx"].shape
        return cls(L.PR_SRC_BUMP2D, nb, 1, nsteps, t)

    @classmethod
    def none(cls) -> "SourceTerm":
        return cls(L.PR_SRC_NONE, 0, 1, 0, {})


class Comm:
    """A pr_comm (include/pr.h "distribution"): NCCL over one process per GPU,
    or `world` in-process virtual ranks on one GPU (one host thread each)."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep            # the local group: destroyed with its last rank
        r, w = ctypes.c_int(), ctypes.c_int()
        check(L.lib().pr_comm_info(self._h, ctypes.byref(r), ctypes.byref(w)), "pr_comm_info")
        self.rank, self.world = r.value, w.value

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(L.lib().pr_comm_nccl_unique_id(buf), "pr_comm_nccl_unique_id")
        return buf.raw

    @classmethod
    def nccl(cls, rank: int, world: int, uid: bytes) -> "Comm":
        assert len(uid) == 128
        h = ctypes.c_void_p()
        check(L.lib().pr_comm_create_nccl(int(rank), int(world), ctypes.create_string_buffer(uid, 128),
                                          ctypes.byref(h)), "pr_comm_create_nccl")
        return cls(h)

    @classmethod
    def local(cls, world: int) -> list:
        hs = (ctypes.c_void_p * world)()
        check(L.lib().pr_comm_create_local(int(world), hs), "pr_comm_create_local")
        return [cls(ctypes.c_void_p(hs[r])) for r in range(world)]

    def close(self):
        if self._h:
            L.lib().pr_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Coarse:
    """Spectral coarse solvers G_q' = U_q Sigma_q V_q^T of the owned intervals."""

    def __init__(self, handle, comm=None, N_total: int = None):
        self._h = handle
        self._comm = comm            # keeps the communicator alive as long as the handle
        self.N_total = N_total

    @classmethod
    def build(cls, op: Operator, N_total: int, m: int, k: int, p: int, seed: int,
              first_interval: int = 0, n_local: int = None, comm: "Comm" = None,
              stream=None, power_iterations: int = 0, independent_adjoint: bool = False) -> "Coarse":
        if n_local is None:
            n_local = N_total - first_interval
        h = ctypes.c_void_p()
        opts = None
        if power_iterations or independent_adjoint:
            opts = ctypes.byref(L.RsvdOpts(int(power_iterations), 1 if independent_adjoint else 0))
        check(L.lib().pr_build_coarse(op._h, int(N_total), int(first_interval), int(n_local),
                                      int(m), int(k), int(p), ctypes.c_uint64(int(seed)), opts,
                                      comm._h if comm is not None else None,
                                      _stream(stream), ctypes.byref(h)), "pr_build_coarse")
        return cls(h, comm, int(N_total))

    @classmethod
    def build_adaptive(cls, op: Operator, N_total: int, m: int, k: int, p0: int, p_max: int, tol: float,
                       seed: int, r: int = 10, first_interval: int = 0, n_local: int = None,
                       comm: "Comm" = None, stream=None):
        """pr_build_coarse_adaptive: returns (Coarse, p_used)."""
        if n_local is None:
            n_local = N_total - first_interval
        h = ctypes.c_void_p()
        pu = ctypes.c_int()
        check(L.lib().pr_build_coarse_adaptive(op._h, int(N_total), int(first_interval), int(n_local), int(m),
                                               int(k), int(p0), int(p_max), float(tol), int(r),
                                               ctypes.c_uint64(int(seed)), None,
                                               comm._h if comm is not None else None, _stream(stream),
                                               ctypes.byref(h), ctypes.byref(pu)), "pr_build_coarse_adaptive")
        return cls(h, comm, int(N_total)), pu.value

    def estimate(self, op: Operator, r: int = 10, seed: int = 0, stream=None) -> np.ndarray:
        """pr_coarse_estimate: per-interval estimate of ||F_q' - G_q'||."""
        est = np.zeros(self.info(raise_on_error=False)["n_local"])
        check(L.lib().pr_coarse_estimate(self._h, op._h, int(r), ctypes.c_uint64(int(seed)), _hptr(est),
                                         _stream(stream)), "pr_coarse_estimate")
        return est

    def info(self, raise_on_error: bool = True) -> dict:
        k, l, nl, first, m = (ctypes.c_int() for _ in range(5))
        delta, eps = ctypes.c_double(), ctypes.c_double()
        st0 = L.lib().pr_coarse_info(self._h, ctypes.byref(k), ctypes.byref(l), ctypes.byref(nl),
                                     ctypes.byref(first), ctypes.byref(m), None, None, None, None)
        if st0 in (L.PR_EINVAL, L.PR_ECUDA):
            check(st0, "pr_coarse_info")
        sig = np.zeros(nl.value * l.value)
        passes = (ctypes.c_int * 2)()
        st = L.lib().pr_coarse_info(self._h, None, None, None, None, None, ctypes.byref(delta),
                                    ctypes.byref(eps), _hptr(sig), passes)
        if raise_on_error and st not in (L.PR_OK, L.PR_EUNAVAIL):
            check(st, "pr_coarse_info")
        return dict(k=k.value, l=l.value, n_local=nl.value, first_interval=first.value, m=m.value,
                    N_total=self.N_total,
                    delta=delta.value, eps=eps.value, sigma=sig.reshape(nl.value, l.value),
                    qr_passes=(passes[0], passes[1]), status=st)

    def apply(self, q_local: int, X, Y, dim: int, stream=None):
        nvec = X.shape[1] if dim == 1 else X.shape[0]
        check(L.lib().pr_coarse_apply(self._h, int(q_local), int(nvec), _ptr(X), _ld(X, dim),
                                      _ptr(Y), _ld(Y, dim), _stream(stream)), "pr_coarse_apply")
        return Y

    # ---- distributed building blocks (include/pr.h) ----
    def sweep_matrices(self, U_prev=None, stream=None):
        check(L.lib().pr_coarse_sweep_matrices(self._h, _ptr(U_prev), _stream(stream)),
              "pr_coarse_sweep_matrices")

    def export(self, U=None, V=None, sigma=None, C=None, stream=None):
        check(L.lib().pr_coarse_export(self._h, _ptr(U), _ptr(V), _ptr(sigma), _ptr(C),
                                       _stream(stream)), "pr_coarse_export")

    def export_interval(self, q_local: int, U_q=None, V_q=None, stream=None):
        check(L.lib().pr_coarse_export_interval(self._h, int(q_local), _ptr(U_q), _ptr(V_q),
                                                _stream(stream)), "pr_coarse_export_interval")

    def project(self, nsrc: int, Y1, Y2, ld: int, d, stream=None):
        check(L.lib().pr_coarse_project(self._h, int(nsrc), _ptr(Y1), _ptr(Y2), int(ld), _ptr(d),
                                        _stream(stream)), "pr_coarse_project")

    def expand(self, nsrc: int, Fu, e, out, ld: int, upd=None, stream=None):
        check(L.lib().pr_coarse_expand(self._h, int(nsrc), _ptr(Fu), _ptr(e), _ptr(out), int(ld),
                                       _ptr(upd), _stream(stream)), "pr_coarse_expand")

    def close(self):
        if self._h:
            L.lib().pr_coarse_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def parareal(G: Coarse, op: Operator, u0, source: SourceTerm, K: int, U_out, nsrc: int = 1,
             hist=None, stream=None):
    """Returns (upd[K, N+1, nsrc], bnorm[N+1, nsrc]) host arrays (all
    boundaries); U_out holds u^K of the handle's boundaries (all of them, or
    the rank's shard + halo block when G was built with a communicator)."""
    Np1 = G.N_total + 1
    upd = np.zeros((max(K, 0), Np1, nsrc))
    bn = np.zeros((Np1, nsrc))
    hs = int(hist.stride(0)) if hist is not None else 0
    check(L.lib().pr_parareal(G._h, op._h, int(nsrc), _ptr(u0),
                              _ld(u0, op.dim) if u0 is not None else 0,
                              ctypes.byref(source.struct), int(K), _ptr(U_out), _ld(U_out, op.dim),
                              _hptr(upd) if K > 0 else None, _hptr(bn),
                              _ptr(hist) if hist is not None else None, hs, _stream(stream)),
          "pr_parareal")
    return upd, bn


def parareal_tol(G: Coarse, op: Operator, u0, source: SourceTerm, K_max: int, tol: float, U_out,
                 nsrc: int = 1, hist=None, stream=None):
    """pr_parareal_tol: a posteriori stopping.  Returns (k_done, upd[k_done,
    N+1, nsrc], bnorm[N+1, nsrc])."""
    Np1 = G.N_total + 1
    upd = np.zeros((max(K_max, 1), Np1, nsrc))
    bn = np.zeros((Np1, nsrc))
    kd = ctypes.c_int()
    hs = int(hist.stride(0)) if hist is not None else 0
    check(L.lib().pr_parareal_tol(G._h, op._h, int(nsrc), _ptr(u0), _ld(u0, op.dim),
                                  ctypes.byref(source.struct), int(K_max), float(tol), _ptr(U_out),
                                  _ld(U_out, op.dim), _hptr(upd), _hptr(bn),
                                  _ptr(hist) if hist is not None else None, hs, ctypes.byref(kd),
                                  _stream(stream)), "pr_parareal_tol")
    return kd.value, upd[:kd.value], bn


def sequential(op: Operator, u0, source: SourceTerm, N: int, m: int, U_out, nsrc: int = 1, stream=None):
    """pr_sequential: u_0 = u0, u_{q+1} = F_{q+1} u_q into U_out ((N+1)*nsrc vectors)."""
    check(L.lib().pr_sequential(op._h, int(nsrc), _ptr(u0), _ld(u0, op.dim), ctypes.byref(source.struct),
                                int(N), int(m), _ptr(U_out), _ld(U_out, op.dim), _stream(stream)),
          "pr_sequential")
    return U_out


def trajectory_error(op: Operator, U, Uref, N: int, m: int, nsrc: int = 1, stream=None):
    """pr_trajectory_error: (err[nsrc], per_interval[N, nsrc]) host arrays."""
    err = np.zeros(nsrc)
    ivl = np.zeros((N, nsrc))
    check(L.lib().pr_trajectory_error(op._h, int(nsrc), int(N), int(m), _ptr(U), _ld(U, op.dim),
                                      _ptr(Uref), _ld(Uref, op.dim), _hptr(err), _hptr(ivl),
                                      _stream(stream)), "pr_trajectory_error")
    return err, ivl


def efficiency(delta: float, eps: float, upd: np.ndarray, traj_err: np.ndarray):
    """pr_efficiency (eq. def_efficiency): upd (K, N+1), traj_err (K+1,) -> eta (K,)."""
    upd = np.ascontiguousarray(upd, dtype=np.float64)
    te = np.ascontiguousarray(traj_err, dtype=np.float64)
    K, Np1 = upd.shape
    eta = np.zeros(K)
    check(L.lib().pr_efficiency(float(delta), float(eps), Np1 - 1, K, _hptr(upd), _hptr(te), _hptr(eta)),
          "pr_efficiency")
    return eta


def parareal_classical(coarse, coarse_source, op: Operator, u0, source: SourceTerm, N: int, m: int, K: int,
                       U_out, nsrc: int = 1, hist=None, stream=None):
    """pr_parareal_classical: coarse = Operator (one backward-Euler step per
    interval, source coarse_source) or None (G = 0).  Returns upd[K, N+1, nsrc]."""
    upd = np.zeros((max(K, 1), N + 1, nsrc))
    hs = int(hist.stride(0)) if hist is not None else 0
    check(L.lib().pr_parareal_classical(coarse._h if coarse is not None else None,
                                        ctypes.byref(coarse_source.struct) if coarse_source is not None else None,
                                        op._h, int(nsrc), _ptr(u0), _ld(u0, op.dim), ctypes.byref(source.struct),
                                        int(N), int(m), int(K), _ptr(U_out), _ld(U_out, op.dim),
                                        _hptr(upd), _ptr(hist) if hist is not None else None, hs,
                                        _stream(stream)), "pr_parareal_classical")
    return upd[:K]


def bounds(delta: float, eps: float, bnorm: np.ndarray, upd: np.ndarray):
    """bnorm: (N+1,), upd: (K, N+1) -> dict of a priori / a posteriori bounds."""
    bnorm = np.ascontiguousarray(bnorm, dtype=np.float64)
    upd = np.ascontiguousarray(upd, dtype=np.float64)
    N = bnorm.shape[0] - 1
    K = upd.shape[0]
    apri = np.zeros((K + 1, N + 1))
    apost = np.zeros((max(K, 1), N + 1))
    sup = np.zeros(max(K, 1))
    check(L.lib().pr_bounds(float(delta), float(eps), N, K, _hptr(bnorm),
                            _hptr(upd) if K > 0 else None, _hptr(apri),
                            _hptr(apost) if K > 0 else None, _hptr(sup) if K > 0 else None),
          "pr_bounds")
    return dict(apriori=apri, apost=apost[:K], apost_sup=sup[:K])


def profile(enable: bool = True):
    check(L.lib().pr_profile(1 if enable else 0), "pr_profile")


def counters(reset: bool = False) -> dict:
    """Kernel launches of the library, and stepper launches / device ms /
    DOF-steps timed with CUDA events while profiling was enabled."""
    kl, sl = ctypes.c_long(), ctypes.c_long()
    ms, dof, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(L.lib().pr_counters(1 if reset else 0, ctypes.byref(kl), ctypes.byref(sl),
                              ctypes.byref(ms), ctypes.byref(dof), ctypes.byref(fl)), "pr_counters")
    return dict(kernel_launches=kl.value, stepper_launches=sl.value, stepper_ms=ms.value,
                stepper_dof_steps=dof.value, stepper_flops=fl.value)


PHASES = ("direct", "build", "offsets", "iteration")


def phase_counters(reset: bool = False) -> dict:
    """Timed fine-propagation launches per phase (pr_phase_counters)."""
    n = (ctypes.c_long * 4)()
    ms = (ctypes.c_double * 4)()
    dof = (ctypes.c_double * 4)()
    check(L.lib().pr_phase_counters(1 if reset else 0, n, ms, dof), "pr_phase_counters")
    return {name: dict(launches=n[i], ms=ms[i], dof_steps=dof[i]) for i, name in enumerate(PHASES)}


def reduced_sweep(C, d, N: int, k: int, nsrc: int, e, stream=None):
    check(L.lib().pr_reduced_sweep(_ptr(C), _ptr(d), int(N), int(k), int(nsrc), _ptr(e),
                                   _stream(stream)), "pr_reduced_sweep")
