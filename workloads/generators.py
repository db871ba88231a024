"""Seeded synthetic inputs for C1..C5 (problem data only, no method arithmetic).

Everything here is *input* to the method of arXiv 2508.08873: the spatial
finite-difference operator A (the paper's fine solver takes the discretized
PDE as given), the initial value u0 and the source term f sampled on
the grid and at the step times.  Both the oracle and the CUDA path receive the
bit-identical arrays produced here, so parity tests compare the methods, not
the samplers.

Conventions:
  * interior points only, h = 1/(n+1), x_i = (i+1) h for i = 0..n-1;
  * global step index g = (interval-1)*m + j, j = 1..m, time t_g = g*dt
    (integer-derived, Z3); the source of step g is evaluated at t_g;
  * 1D source: f_s(x_i, t_g) = sum_r amp[s, r] * space[r, i] * time[r, g-1];
  * 2D source: f(x_i, y_j, t_g) = sum_b gx[b, g-1, i] * gy[b, g-1, j].
"""
from __future__ import annotations

import numpy as np

from .configs import Config

BETA_CD = 20.0      # advection speed of the test-only convection_diffusion operator


# --------------------------------------------------------------------------- grid
def grid_1d(n: int) -> np.ndarray:
    h = 1.0 / (n + 1)
    return (np.arange(n, dtype=np.float64) + 1.0) * h


def step_times(cfg: Config) -> np.ndarray:
    """t_g for g = 1..N*m (index g-1), from the integer step index (Z3)."""
    g = np.arange(1, cfg.N * cfg.m + 1, dtype=np.float64)
    return g * cfg.dt


# ------------------------------------------------------------------- operator A
def operator_1d(cfg: Config):
    """Tridiagonal FD matrix A (so that u_t = -A u + f) as (sub, diag, sup).

    sub[i] = A[i, i-1] (sub[0] unused = 0), sup[i] = A[i, i+1] (sup[n-1] = 0).
    heat (C1, C2):            A = tridiag(-1, 2, -1) / h^2                (Z2)
    reaction_diffusion (C4):  A u = -(kappa u_x)_x + 0.5 u, kappa at the
                              midpoints x_{i+-1/2}, conservative form    (Z2)
    convection_diffusion (test-only T4N / C4N, non-symmetric):
                              C4's operator plus beta u_x, beta = 20, upwind
                              (u_i - u_{i-1}) / h -- an M-matrix with A != A^T,
                              so F' is not normal and F'^* != F' (the regime
                              of Exp 2)
    """
    n, h = cfg.n, cfg.h
    if cfg.problem == "heat":
        sub = np.full(n, -1.0 / (h * h))
        sup = np.full(n, -1.0 / (h * h))
        diag = np.full(n, 2.0 / (h * h))
    elif cfg.problem == "reaction_diffusion":
        # kappa(x) = 1 + 0.5 sin(2 pi x) (BJ C4) at x_{i-1/2}, i = 0..n  (n+1 faces)
        xf = (np.arange(n + 1, dtype=np.float64) + 0.5) * h
        kap = 1.0 + 0.5 * np.sin(2.0 * np.pi * xf)
        km, kp = kap[:-1], kap[1:]          # kappa_{i-1/2}, kappa_{i+1/2}
        diag = (km + kp) / (h * h) + 0.5
        sub = -km / (h * h)
        sup = -kp / (h * h)
    elif cfg.problem == "convection_diffusion":
        xf = (np.arange(n + 1, dtype=np.float64) + 0.5) * h
        kap = 1.0 + 0.5 * np.sin(2.0 * np.pi * xf)
        km, kp = kap[:-1], kap[1:]
        diag = (km + kp) / (h * h) + BETA_CD / h + 0.5
        sub = -km / (h * h) - BETA_CD / h
        sup = -kp / (h * h)
    else:
        raise ValueError(cfg.problem)
    sub = sub.copy()
    sup = sup.copy()
    sub[0] = 0.0
    sup[-1] = 0.0
    return sub, diag, sup


def operator_1d_sums(cfg: Config):
    """Exact row and column sums of A, from the problem definition (not by
    adding the stencil entries, which cancels): interior rows of the heat
    operator sum to 0, of C4 to the reaction coefficient 0.5; the first/last
    rows keep the coupling to the eliminated Dirichlet boundary value.
    A is symmetric here, so the column sums equal the row sums."""
    n, h = cfg.n, cfg.h
    if cfg.problem == "heat":
        rs = np.zeros(n)
        rs[0] += 1.0 / (h * h)
        rs[-1] += 1.0 / (h * h)
    elif cfg.problem == "reaction_diffusion":
        xf = (np.arange(n + 1, dtype=np.float64) + 0.5) * h
        kap = 1.0 + 0.5 * np.sin(2.0 * np.pi * xf)
        rs = np.full(n, 0.5)
        rs[0] += kap[0] / (h * h)
        rs[-1] += kap[-1] / (h * h)
    elif cfg.problem == "convection_diffusion":
        # interior rows and columns sum to the reaction coefficient 0.5 (the
        # advection stencil -beta/h, +beta/h cancels in both directions); the
        # boundary rows / columns keep the eliminated Dirichlet couplings
        xf = (np.arange(n + 1, dtype=np.float64) + 0.5) * h
        kap = 1.0 + 0.5 * np.sin(2.0 * np.pi * xf)
        rs = np.full(n, 0.5)
        rs[0] += kap[0] / (h * h) + BETA_CD / h
        rs[-1] += kap[-1] / (h * h)
        cs = np.full(n, 0.5)
        cs[0] += kap[0] / (h * h)
        cs[-1] += kap[-1] / (h * h) + BETA_CD / h
        return rs, cs
    else:
        raise ValueError(cfg.problem)
    return rs, rs.copy()


def laplacian_1d_for_2d(cfg: Config):
    """The 1D factor T = tridiag(-1,2,-1)/h^2 of the 2D 5-point A = T(x)I + I(x)T."""
    n, h = cfg.n, cfg.h
    sub = np.full(n, -1.0 / (h * h))
    sup = np.full(n, -1.0 / (h * h))
    diag = np.full(n, 2.0 / (h * h))
    sub[0] = 0.0
    sup[-1] = 0.0
    return sub, diag, sup


def laplacian_1d_for_2d_sums(cfg: Config):
    """Exact row sums of T (0 inside, 1/h^2 on the two boundary rows)."""
    rs = np.zeros(cfg.n)
    rs[0] = rs[-1] = 1.0 / (cfg.h * cfg.h)
    return rs


# ------------------------------------------------------------------------ u0
def initial_value(cfg: Config) -> np.ndarray:
    """u0 on the interior grid: shape (n,) in 1D, (n, n) [x-index, y-index] in 2D."""
    if cfg.u0 == "exp2":                           # 10 chi_[0.6, 0.8] (workloads/exp2.py)
        from . import exp2
        return exp2.initial_value(cfg.n)
    rng = np.random.default_rng(cfg.seed_u0)
    if cfg.dim == 1:
        x = grid_1d(cfg.n)
        if cfg.u0 == "x1mx":                       # C1, and C4 by Z13
            return x * (1.0 - x)
        if cfg.u0 == "sine20":                     # C2, Z16
            a = rng.standard_normal(20)
            u = np.zeros(cfg.n)
            for j in range(1, 21):
                u += (a[j - 1] / j) * np.sin(j * np.pi * x)
            return u
        raise ValueError(cfg.u0)
    if cfg.u0 == "smooth2d":                       # C3, C5, Z15
        n = cfg.n
        u = np.zeros((n + 2, n + 2))
        u[1:-1, 1:-1] = rng.standard_normal((n, n))
        for _ in range(10):                        # 10 Jacobi sweeps, omega = 1, zero boundary
            v = np.zeros_like(u)
            v[1:-1, 1:-1] = 0.25 * (u[:-2, 1:-1] + u[2:, 1:-1] + u[1:-1, :-2] + u[1:-1, 2:])
            u = v
        return np.ascontiguousarray(u[1:-1, 1:-1])
    raise ValueError(cfg.u0)


# ---------------------------------------------------------------------- source
def source_1d(cfg: Config):
    """Separable sampled source: (space[R, n], time[R, N*m], amp[nsrc, R])."""
    if cfg.source == "exp2":                       # Exp 2 (workloads/exp2.py)
        from . import exp2
        return exp2.source(cfg.problem, cfg.n, cfg.T, cfg.N * cfg.m, cfg.nsrc)
    x = grid_1d(cfg.n)
    t = step_times(cfg)
    if cfg.source == "c1":                         # f = sin(pi x) cos(2 pi t)
        space = np.sin(np.pi * x)[None, :]
        time = np.cos(2.0 * np.pi * t)[None, :]
        amp = np.ones((cfg.nsrc, 1))
    elif cfg.source == "c2":                       # f = exp(-100 (x-0.5)^2) sin(10 t)
        space = np.exp(-100.0 * (x - 0.5) ** 2)[None, :]
        time = np.sin(10.0 * t)[None, :]
        amp = np.ones((cfg.nsrc, 1))
    elif cfg.source == "c4":                       # f_s = sum_{j<=8} a_{s,j} sin(j pi x) cos(j t), Z17
        rng = np.random.default_rng(cfg.seed_src)
        J = np.arange(1, 9, dtype=np.float64)
        space = np.sin(np.pi * J[:, None] * x[None, :])
        time = np.cos(J[:, None] * t[None, :])
        amp = rng.standard_normal((cfg.nsrc, 8))
    else:
        raise ValueError(cfg.source)
    return (np.ascontiguousarray(space), np.ascontiguousarray(time),
            np.ascontiguousarray(amp))


def bump_centers(cfg: Config, nb: int):
    """c_b(t) = (0.5 + 0.25 cos(2 pi t/T + b pi/2), 0.5 + 0.25 sin(...)), Z14."""
    t = step_times(cfg)
    cx = np.empty((nb, t.size))
    cy = np.empty((nb, t.size))
    for b in range(nb):
        ph = 2.0 * np.pi * t / cfg.T + b * np.pi / 2.0
        cx[b] = 0.5 + 0.25 * np.cos(ph)
        cy[b] = 0.5 + 0.25 * np.sin(ph)
    return cx, cy


def source_2d(cfg: Config):
    """Moving Gaussian bumps, separable in x and y (Z14):
    f(x, y, t_g) = sum_b gx[b, g-1, i] * gy[b, g-1, j],
    gx = 100 exp(-(x - cx)^2 / (2 s^2)), gy = exp(-(y - cy)^2 / (2 s^2)), s = 0.05.
    """
    nb = {"bump1": 1, "bump4": 4}[cfg.source]
    x = grid_1d(cfg.n)
    cx, cy = bump_centers(cfg, nb)
    s2 = 2.0 * 0.05 ** 2
    gx = 100.0 * np.exp(-((x[None, None, :] - cx[:, :, None]) ** 2) / s2)
    gy = np.exp(-((x[None, None, :] - cy[:, :, None]) ** 2) / s2)
    return np.ascontiguousarray(gx), np.ascontiguousarray(gy)


# ------------------------------------------------------------ layout helpers
def pad2d(u: np.ndarray) -> np.ndarray:
    """(…, n, n) interior field -> (…, n+1, n+1) with a zero ghost row/col 0.

    This is the storage layout of the CUDA 2D path (index 0 is the Dirichlet
    boundary, always zero); pure data movement.
    """
    n = u.shape[-1]
    out = np.zeros(u.shape[:-2] + (n + 1, n + 1), dtype=np.float64)
    out[..., 1:, 1:] = u
    return out


def unpad2d(u: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(u[..., 1:, 1:])


def pad1d_last(v: np.ndarray) -> np.ndarray:
    """(…, n) -> (…, n+1) with a zero at index 0 (2D source factors)."""
    out = np.zeros(v.shape[:-1] + (v.shape[-1] + 1,), dtype=np.float64)
    out[..., 1:] = v
    return out
