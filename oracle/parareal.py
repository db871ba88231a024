"""Parareal with spectral coarse solvers -- TEST INFRASTRUCTURE ONLY.

Direct form of eq. def_Parareal:
    u^k_0 := u_0,   u^0_{n+1} := G_{n+1} u^0_n,
    u^{k+1}_{n+1} := F_{n+1} u^k_n + G_{n+1} u^{k+1}_n - G_{n+1} u^k_n,
with G_n v = G_n' v + b_n (eq. spectral_G) and b_n = F_n 0
(eq. F_n_affine).  Update norms ||u^k_n - u^{k-1}_n|| feed the
a posteriori bound.  Several sources share G_n' and differ in
b_n (Remark affine_g_n).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fine import fine


@dataclass
class PararealResult:
    U: np.ndarray        # (K+1, N+1, nvec, ...) all iterates u^k_n
    b: np.ndarray        # (N+1, nvec, ...) offsets b_n (b_0 unused = u0 for bounds)
    upd: np.ndarray      # (K+1, N+1, nvec) ||u^k_n - u^{k-1}_n||  (row 0 = 0)


def offsets(op, N: int, nvec_shape, src, src_index=None):
    """b_n = F_n 0 for n = 1..N (one vector per source)."""
    zero = np.zeros(nvec_shape)
    return np.stack([np.zeros(nvec_shape)] +
                    [fine(op, n, zero, "affine", src, src_index) for n in range(1, N + 1)])


def parareal(op, truncs, u0: np.ndarray, N: int, K: int, src, src_index=None) -> PararealResult:
    """u0: (nvec, ...) one initial value per source.  truncs[n-1] is G_n'."""
    u0 = np.asarray(u0, dtype=np.float64)
    shp = u0.shape
    flat = lambda x: x.reshape(shp[0], -1)

    def G(n, x, b):                      # G_n x = G_n' x + b_n
        return truncs[n - 1].apply_linear(flat(x)).reshape(shp) + b[n]

    b = offsets(op, N, shp, src, src_index)
    U = np.zeros((K + 1, N + 1) + shp)
    upd = np.zeros((K + 1, N + 1, shp[0]))
    U[0, 0] = u0
    for n in range(N):                                 # initialization
        U[0, n + 1] = G(n + 1, U[0, n], b)
    for k in range(K):
        Fu = [fine(op, n + 1, U[k, n], "affine", src, src_index) for n in range(N)]
        Gold = [G(n + 1, U[k, n], b) for n in range(N)]
        U[k + 1, 0] = u0
        for n in range(N):                             # sequential sweep
            U[k + 1, n + 1] = Fu[n] + G(n + 1, U[k + 1, n], b) - Gold[n]
        d = (U[k + 1] - U[k]).reshape((N + 1) * shp[0], -1)
        upd[k + 1] = np.linalg.norm(d, axis=1).reshape(N + 1, shp[0])
    return PararealResult(U=U, b=b, upd=upd)


def parareal_classical(op, Gfun, u0: np.ndarray, N: int, K: int, src, src_index=None) -> PararealResult:
    """eq. def_Parareal with an arbitrary coarse solver Gfun(n, x) = G_n x
    (affine; e.g. one coarse backward-Euler step, or 0)."""
    u0 = np.asarray(u0, dtype=np.float64)
    shp = u0.shape
    U = np.zeros((K + 1, N + 1) + shp)
    upd = np.zeros((K + 1, N + 1, shp[0]))
    U[0, 0] = u0
    for n in range(N):
        U[0, n + 1] = Gfun(n + 1, U[0, n])
    for k in range(K):
        Fu = [fine(op, n + 1, U[k, n], "affine", src, src_index) for n in range(N)]
        Gold = [Gfun(n + 1, U[k, n]) for n in range(N)]
        U[k + 1, 0] = u0
        for n in range(N):
            U[k + 1, n + 1] = Gfun(n + 1, U[k + 1, n]) + Fu[n] - Gold[n]
        d = (U[k + 1] - U[k]).reshape((N + 1) * shp[0], -1)
        upd[k + 1] = np.linalg.norm(d, axis=1).reshape(N + 1, shp[0])
    return PararealResult(U=U, b=np.zeros((N + 1,) + shp), upd=upd)


def trajectory_error(op, Uk: np.ndarray, Uref: np.ndarray, N: int, src, src_index=None):
    """max over t in [0, T] of ||u^k(t) - u(t)||: inside
    [t_{n-1}, t_n) both are the fine trajectories (one step at a time, with the
    source) started from u^k_{n-1} and u_{n-1}; t = T is the end of interval
    N's (reading R-TRAJ).  Uk, Uref: (N+1, nvec, n).  Returns (nvec,)."""
    from .fine import fine_trajectory
    best = np.zeros(Uk.shape[1])
    for n in range(1, N + 1):
        a = fine_trajectory(op, n, Uk[n - 1], src, src_index)
        b = fine_trajectory(op, n, Uref[n - 1], src, src_index)
        last = len(a) if n == N else len(a) - 1
        for j in range(last):
            best = np.maximum(best, np.linalg.norm((a[j] - b[j]).reshape(a[j].shape[0], -1), axis=1))
    return best
