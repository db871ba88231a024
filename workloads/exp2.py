"""Problem data of the paper's Experiment 2 (eq. ex2) -- inputs only.

    u_t - d/dx[(1 + 0.9 sin(7 pi t + 2 pi x)) u_x] = f(x, t),   x in (0, 1), t in [0, 1]
    u_x(0, t) = u_x(1, t) = 0  (Neumann),   f = 100 sin(5 pi t) (1 + cos(3 pi x))  (eq. oned_heat)
    u(x, 0) = u_0 = 10 chi_[0.6, 0.8]  (nodal interpolation, reading R-E2)

Like every module under workloads/, this holds NO arithmetic of the method (no
solves, no time stepping): it assembles the step matrices and load vectors the
fine solver consumes.  Both the oracle and the CUDA path read it.

Two discretisations on the uniform mesh x_i = i h, h = 1/(n-1), i = 0..n-1
(all nodes are unknowns with Neumann conditions):

* "exp2_fem" -- linear finite elements, as in the paper: consistent
  mass matrix M (h/6, 2h/3, h/6; h/3 at the boundary nodes) and stiffness
  A(t) with the element conductivity kappa evaluated at the element midpoint at
  time t (midpoint rule).  Step g (implicit Euler, t_g = g dt):
        (M + dt A(t_g)) u_g = M u_{g-1} + dt l(t_g),   l_i(t) = int f(x, t) phi_i dx.
* "exp2_fd" -- finite differences with mirrored ghost nodes at the Neumann
  boundary: A(t) = D^{-1} K(t) with K the same stiffness and D = diag(h, ..,
  h/2 at the ends) / h, M = I.  A(t) is NOT symmetric (the boundary rows are
  doubled), so every step is a non-symmetric tridiagonal solve.

In both, A(t) 1 = 0 (no flux through the boundary), so F_n' 1 = 1 for every
interval: the constant mode is undamped and delta = max sigma_{n,1} >= 1
(P:511-513).
"""
from __future__ import annotations

import numpy as np


def kappa(x, t):
    return 1.0 + 0.9 * np.sin(7.0 * np.pi * t + 2.0 * np.pi * x)


def nodes(n: int) -> np.ndarray:
    return np.linspace(0.0, 1.0, n)


def step_times(T: float, nsteps: int) -> np.ndarray:
    """t_g = g dt, g = 1..nsteps (implicit Euler evaluates at the new time, Z3)."""
    dt = T / nsteps
    return dt * np.arange(1, nsteps + 1, dtype=np.float64)


def stiffness(n: int, t: float):
    """K(t) = (sub, diag, sup), element-midpoint conductivity; rows sum to 0."""
    h = 1.0 / (n - 1)
    xm = (np.arange(n - 1) + 0.5) * h            # element midpoints
    ke = kappa(xm, t) / h                         # element stiffness kappa_e / h
    sub = np.zeros(n)
    sup = np.zeros(n)
    diag = np.zeros(n)
    sub[1:] = -ke
    sup[:-1] = -ke
    diag[:-1] += ke
    diag[1:] += ke
    return sub, diag, sup


def mass(n: int):
    """Consistent P1 mass matrix (sub, diag, sup); row sums int phi_i dx."""
    h = 1.0 / (n - 1)
    sub = np.full(n, h / 6.0)
    sup = np.full(n, h / 6.0)
    sub[0] = 0.0
    sup[-1] = 0.0
    diag = np.full(n, 2.0 * h / 3.0)
    diag[0] = diag[-1] = h / 3.0
    rows = np.full(n, h)
    rows[0] = rows[-1] = h / 2.0
    return sub, diag, sup, rows


def step_matrices(problem: str, n: int, T: float, nsteps: int):
    """Left-hand sides L_g = M + dt A(t_g) for g = 1..nsteps as (nsteps, n)
    arrays (sub, diag, sup), their exact row sums (the row sums of M, since
    A 1 = 0), and M (None for the FD variant)."""
    dt = T / nsteps
    ts = step_times(T, nsteps)
    sub = np.empty((nsteps, n))
    diag = np.empty((nsteps, n))
    sup = np.empty((nsteps, n))
    if problem == "exp2_fem":
        ms, md, mp, mrow = mass(n)
        for g, t in enumerate(ts):
            a, d, c = stiffness(n, t)
            sub[g] = ms + dt * a
            diag[g] = md + dt * d
            sup[g] = mp + dt * c
        rowsum = np.tile(mrow, (nsteps, 1))
        return (sub, diag, sup), rowsum, (ms, md, mp)
    if problem == "exp2_fd":
        dscale = np.ones(n)
        dscale[0] = dscale[-1] = 0.5               # lumped mass / h at the boundary nodes
        h = 1.0 / (n - 1)
        for g, t in enumerate(ts):
            a, d, c = stiffness(n, t)
            sub[g] = dt * a / (h * dscale)
            diag[g] = 1.0 + dt * d / (h * dscale)
            sup[g] = dt * c / (h * dscale)
        return (sub, diag, sup), np.ones((nsteps, n)), None
    raise ValueError(problem)


def load_space(problem: str, n: int) -> np.ndarray:
    """Spatial factor of f = 100 sin(5 pi t) (1 + cos(3 pi x)): for FEM the load
    vector int (1 + cos(3 pi x)) phi_i dx (exact for the hat functions), for FD
    the nodal values."""
    x = nodes(n)
    if problem == "exp2_fd":
        return 1.0 + np.cos(3.0 * np.pi * x)
    h = 1.0 / (n - 1)
    k = 3.0 * np.pi
    # int cos(k x) phi_i dx, exact: interior hats 2 (1 - cos kh) / (k^2 h) cos(k x_i);
    # half hats int_0^h cos(kx)(1 - x/h) dx = (1 - cos kh)/(k^2 h) and
    # int_{1-h}^1 cos(kx)(x - 1 + h)/h dx = (cos k - cos k(1-h))/(k^2 h) + sin(k)/k
    c = (1.0 - np.cos(k * h)) / (k * k * h)
    b = 2.0 * c * np.cos(k * x)
    b[0] = c
    b[-1] = (np.cos(k) - np.cos(k * (1.0 - h))) / (k * k * h) + np.sin(k) / k
    ones = np.full(n, h)
    ones[0] = ones[-1] = h / 2.0
    return ones + b


def source(problem: str, n: int, T: float, nsteps: int, nsrc: int = 1):
    """(space[1, n], time[1, nsteps], amp[nsrc, 1]) in the PR_SRC_SEP1D form."""
    t = step_times(T, nsteps)
    space = load_space(problem, n)[None, :]
    time = (100.0 * np.sin(5.0 * np.pi * t))[None, :]
    amp = np.ones((nsrc, 1))
    return np.ascontiguousarray(space), np.ascontiguousarray(time), amp


def initial_value(n: int) -> np.ndarray:
    x = nodes(n)
    return np.where((x >= 0.6 - 1e-12) & (x <= 0.8 + 1e-12), 10.0, 0.0)
