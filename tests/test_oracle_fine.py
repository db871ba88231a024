"""Pins for oracle/fine.py: backward-Euler fine solver, affine split
(P:162-167), adjoint.  Each pin compares against something other
than the oracle: dense inverses (numpy.linalg), closed-form spectra (P:708-716,
P:819-821 discrete analog), manufactured solutions."""
from dataclasses import replace

import numpy as np
import pytest

from oracle._clib import thomas_batch
from oracle.fine import Op1D, Op2D, fine, make_op, sequential_reference, sine_matrix
from oracle.rsvd import dense_transfer
from workloads import generators as G
from workloads.configs import C1, C3, C4, get


def test_thomas_manufactured_solution():
    rng = np.random.default_rng(0)
    n, nsys = 301, 17
    sub = rng.uniform(-1, 1, n)
    sup = rng.uniform(-1, 1, n)
    diag = 3.0 + rng.uniform(0, 1, n)
    shift = rng.uniform(0, 2, nsys)
    Xtrue = rng.standard_normal((nsys, n))
    B = np.empty_like(Xtrue)
    for s in range(nsys):
        A = np.diag(diag + shift[s]) + np.diag(sub[1:], -1) + np.diag(sup[:-1], 1)
        B[s] = A @ Xtrue[s]
    X = B.copy()
    thomas_batch(sub, diag, sup, X, shift)
    assert np.max(np.abs(X - Xtrue)) <= 1e-13 * np.max(np.abs(Xtrue))


def _dense_power(T, m):
    Ti = np.linalg.inv(T)
    return np.linalg.matrix_power(Ti, m)


@pytest.mark.parametrize("n,m", [(7, 3), (31, 16), (64, 5)])
def test_1d_linear_matches_dense_power(n, m):
    cfg = replace(C1, n=n, m=m)
    op = make_op(cfg)
    F = dense_transfer(op)
    T = np.eye(n) + cfg.dt * op.dense_A()
    ref = _dense_power(T, m)
    assert np.max(np.abs(F - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_1d_heat_closed_form_spectrum():
    """sigma_j = (1 + dt lam_j)^(-m), lam_j = (4/h^2) sin^2(j pi h / 2): the discrete
    analog of sigma_{R+1} = exp(-(R+1)^2 pi^2 dT)."""
    cfg = C1
    op = make_op(cfg)
    F = dense_transfer(op)
    s = np.linalg.svd(F, compute_uv=False)
    j = np.arange(1, cfg.n + 1)
    lam = 4.0 / cfg.h ** 2 * np.sin(j * np.pi * cfg.h / 2) ** 2
    ref = np.sort((1 + cfg.dt * lam) ** (-cfg.m))[::-1]
    assert np.max(np.abs(s - ref)) <= 1e-14 * ref[0]
    assert abs(s[0] - 0.5413) < 1e-4            # sigma_1(C1)


def test_1d_adjoint_identity_nonsymmetric():
    rng = np.random.default_rng(1)
    n = 40
    sub = -1.0 - rng.uniform(0, 1, n)
    sup = -1.0 - rng.uniform(0, 1, n)
    diag = 4.0 + rng.uniform(0, 1, n)
    sub[0] = 0
    sup[-1] = 0
    op = Op1D(sub, diag, sup, dt=0.3, m=4)
    v = rng.standard_normal((3, n))
    w = rng.standard_normal((3, n))
    Fv = fine(op, 1, v, "linear")
    Fsw = fine(op, 1, w, "adjoint")
    np.testing.assert_allclose(np.sum(Fv * w, 1), np.sum(v * Fsw, 1), rtol=1e-13, atol=0)
    # and against the dense transpose
    Fd = dense_transfer(op)
    np.testing.assert_allclose(dense_transfer(op, mode="adjoint"), Fd.T, rtol=0, atol=1e-14)


def test_1d_affine_with_source_brute_force():
    cfg = replace(get("T4"), n=29, m=5, N=3)
    op = make_op(cfg)
    src = G.source_1d(cfg)
    space, time, amp = src
    rng = np.random.default_rng(2)
    v = rng.standard_normal((cfg.nsrc, cfg.n))
    sidx = np.arange(cfg.nsrc)
    out = fine(op, 2, v, "affine", src, sidx)
    T = np.eye(cfg.n) + cfg.dt * op.dense_A()
    for s in range(cfg.nsrc):
        x = v[s].copy()
        for j in range(1, cfg.m + 1):
            g = 1 * cfg.m + j
            t = g * cfg.dt
            f = sum(amp[s, r] * space[r] * time[r, g - 1] for r in range(space.shape[0]))
            # the C4 source formula itself (Z17), evaluated independently of the sampler
            xg = G.grid_1d(cfg.n)
            rng2 = np.random.default_rng(cfg.seed_src)
            a = rng2.standard_normal((cfg.nsrc, 8))
            f2 = sum(a[s, jj - 1] * np.sin(jj * np.pi * xg) * np.cos(jj * t) for jj in range(1, 9))
            np.testing.assert_allclose(f, f2, rtol=0, atol=1e-12)
            x = np.linalg.solve(T, x + cfg.dt * f)
        np.testing.assert_allclose(out[s], x, rtol=0, atol=1e-12 * np.max(np.abs(x)))


def test_affinity_F_equals_linear_plus_offset():
    cfg = get("T4")
    op = make_op(cfg)
    src = G.source_1d(cfg)
    rng = np.random.default_rng(3)
    v = rng.standard_normal((cfg.nsrc, cfg.n))
    idx = np.arange(cfg.nsrc)
    Fv = fine(op, 3, v, "affine", src, idx)
    lin = fine(op, 3, v, "linear")
    b = fine(op, 3, np.zeros_like(v), "affine", src, idx)
    np.testing.assert_allclose(Fv, lin + b, rtol=0, atol=1e-12 * np.max(np.abs(Fv)))


def test_c4_operator_manufactured_solution():
    """A u ~ -(kappa u')' + 0.5 u to O(h^2) for a smooth u (reading Z2)."""
    errs = []
    for n in (63, 127, 255):
        cfg = replace(C4, n=n)
        sub, diag, sup = G.operator_1d(cfg)
        x = G.grid_1d(n)
        u = np.sin(np.pi * x) * np.exp(x)            # u(0) = u(1) = 0
        Au = diag * u
        Au[1:] += sub[1:] * u[:-1]
        Au[:-1] += sup[:-1] * u[1:]
        up = np.pi * np.cos(np.pi * x) * np.exp(x) + np.sin(np.pi * x) * np.exp(x)
        upp = (-np.pi ** 2 * np.sin(np.pi * x) + 2 * np.pi * np.cos(np.pi * x)
               + np.sin(np.pi * x)) * np.exp(x)
        kap = 1 + 0.5 * np.sin(2 * np.pi * x)
        kp = np.pi * np.cos(2 * np.pi * x)
        exact = -(kp * up + kap * upp) + 0.5 * u
        errs.append(np.max(np.abs(Au - exact)))
    assert errs[0] / errs[1] > 3.5 and errs[1] / errs[2] > 3.5


# ------------------------------------------------------------------ 2D
def test_sine_matrix_diagonalises_T():
    n = 21
    cfg = replace(C3, n=n)
    op = make_op(cfg)
    S = sine_matrix(n)
    np.testing.assert_allclose(S @ S, np.eye(n), atol=1e-14)
    a, d, c = op.A1
    T = np.diag(d) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
    L = S @ T @ S
    np.testing.assert_allclose(L, np.diag(op.lam), atol=1e-12 * np.max(op.lam))


@pytest.mark.parametrize("n,m", [(5, 3), (9, 7)])
def test_2d_linear_matches_dense_power(n, m):
    cfg = replace(C3, n=n, m=m)
    op = make_op(cfg)
    F = dense_transfer(op)
    T = np.eye(n * n) + cfg.dt * op.dense_A()
    ref = _dense_power(T, m)
    assert np.max(np.abs(F - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_2d_affine_with_bumps_brute_force():
    cfg = replace(get("T2D"), n=8, m=4, N=3, source="bump4")
    op = make_op(cfg)
    gx, gy = G.source_2d(cfg)
    rng = np.random.default_rng(4)
    v = rng.standard_normal((cfg.n, cfg.n))
    out = fine(op, 3, v, "affine", (gx, gy))
    T = np.eye(cfg.n ** 2) + cfg.dt * op.dense_A()
    x = v.ravel().copy()
    xg = G.grid_1d(cfg.n)
    for j in range(1, cfg.m + 1):
        g = 2 * cfg.m + j
        t = g * cfg.dt
        f = np.zeros((cfg.n, cfg.n))
        for b in range(4):       # Z14 formula, evaluated independently of the sampler
            ph = 2 * np.pi * t / cfg.T + b * np.pi / 2
            cx, cy = 0.5 + 0.25 * np.cos(ph), 0.5 + 0.25 * np.sin(ph)
            f += 100 * np.exp(-((xg[:, None] - cx) ** 2 + (xg[None, :] - cy) ** 2) / (2 * 0.05 ** 2))
        x = np.linalg.solve(T, x + cfg.dt * f.ravel())
    np.testing.assert_allclose(out.ravel(), x, rtol=0, atol=1e-12 * np.max(np.abs(x)))


def test_2d_closed_form_spectrum_pairs():
    cfg = replace(C3, n=9, m=6)
    op = make_op(cfg)
    s = np.linalg.svd(dense_transfer(op), compute_uv=False)
    j = np.arange(1, cfg.n + 1)
    lam = 4.0 / cfg.h ** 2 * np.sin(j * np.pi * cfg.h / 2) ** 2
    ref = np.sort(((1 + cfg.dt * (lam[:, None] + lam[None, :])) ** (-cfg.m)).ravel())[::-1]
    assert np.max(np.abs(s - ref)) <= 1e-14 * ref[0]


def test_sequential_reference_composes_fine_solves():
    cfg = get("T1")
    op = make_op(cfg)
    src = G.source_1d(cfg)
    u0 = G.initial_value(cfg)[None]
    U = sequential_reference(op, u0, cfg.N, src)
    # one long backward-Euler run over N*m steps equals the composition
    T = np.eye(cfg.n) + cfg.dt * op.dense_A()
    x = u0[0].copy()
    space, time, amp = src
    for g in range(1, cfg.N * cfg.m + 1):
        x = np.linalg.solve(T, x + cfg.dt * amp[0, 0] * space[0] * time[0, g - 1])
    np.testing.assert_allclose(U[-1, 0], x, rtol=0, atol=1e-12 * np.max(np.abs(x)))


def _thomas_longdouble(sub, diag, sup, X):
    """Reference Thomas in x87 extended precision (64-bit mantissa), vectorised
    over systems: rounding 2^-64 instead of 2^-53."""
    L = np.longdouble
    a, d, c = sub.astype(L), np.asarray(diag).astype(L), sup.astype(L)
    x = X.astype(L).T.copy()               # (n, nsys)
    n = x.shape[0]
    cp = np.zeros(n, dtype=L)
    den = d[0]
    cp[0] = c[0] / den
    x[0] = x[0] / den
    for i in range(1, n):
        den = d[i] - a[i] * cp[i - 1]
        cp[i] = (c[i] if i < n - 1 else L(0)) / den
        x[i] = (x[i] - a[i] * x[i - 1]) / den
    for i in range(n - 2, -1, -1):
        x[i] = x[i] - cp[i] * x[i + 1]
    return x.T


def test_rowsum_pivots_are_condition_independent():
    """Reading R-ACC: with pivots from exact row sums the stepper's error stays
    at m*u even for C4's stiffness (dt*kappa/h^2 ~ 2.5e4); textbook pivots give
    the coherent m*u*cond drift."""
    assert np.finfo(np.longdouble).nmant >= 63
    cfg = replace(C4, m=8)
    op = make_op(cfg)
    rng = np.random.default_rng(8)
    x0 = np.abs(rng.standard_normal((2, cfg.n))) + np.sin(np.pi * G.grid_1d(cfg.n))
    # the matrix is defined by its off-diagonals and exact row sums (problem
    # data); its diagonal rowsum - sub - sup is formed in extended precision
    a, _, c = op.T
    L = np.longdouble
    dL = op.T_rs.astype(L) - a.astype(L) - c.astype(L)
    ref = x0.astype(L)
    for _ in range(cfg.m):
        ref = _thomas_longdouble(a, dL, c, ref)
    ref = ref.astype(np.float64)
    acc = fine(op, 1, x0, "linear")
    rel_acc = np.max(np.abs(acc - ref)) / np.max(np.abs(ref))
    plain = x0.copy()
    for _ in range(cfg.m):
        thomas_batch(*op.T, plain)                      # textbook pivots
    rel_plain = np.max(np.abs(plain - ref)) / np.max(np.abs(ref))
    assert rel_acc < 50 * cfg.m * 1.1e-16
    assert rel_plain > 10 * rel_acc


def test_convection_diffusion_operator_and_adjoint_dense():
    """The test-only non-symmetric operator (T4N): the assembled A is the upwind
    convection-diffusion stencil (independently re-evaluated here), its exact
    row / column sums match, and the oracle's F' and F'^* equal the dense
    (I + dt A)^{-m} and its transpose (adjoint = transposed steps in reverse
    order), which differ by far more than rounding."""
    from workloads.generators import BETA_CD
    cfg = replace(get("T4N"), n=40, m=7)
    op = make_op(cfg)
    h = cfg.h
    A = op.dense_A()
    x = G.grid_1d(cfg.n)
    kap = lambda y: 1.0 + 0.5 * np.sin(2.0 * np.pi * y)
    for i in (0, 17, cfg.n - 1):
        km, kp = kap(x[i] - h / 2), kap(x[i] + h / 2)
        assert A[i, i] == pytest.approx((km + kp) / h ** 2 + BETA_CD / h + 0.5, rel=1e-14)
        if i > 0:
            assert A[i, i - 1] == pytest.approx(-km / h ** 2 - BETA_CD / h, rel=1e-14)
        if i < cfg.n - 1:
            assert A[i, i + 1] == pytest.approx(-kp / h ** 2, rel=1e-14)
    rs, cs = G.operator_1d_sums(cfg)
    np.testing.assert_allclose(A.sum(axis=1), rs, rtol=1e-9, atol=1e-9 * np.abs(A).max())
    np.testing.assert_allclose(A.sum(axis=0), cs, rtol=1e-9, atol=1e-9 * np.abs(A).max())
    F = np.linalg.matrix_power(np.linalg.inv(np.eye(cfg.n) + cfg.dt * A), cfg.m)
    X = np.random.default_rng(9).standard_normal((3, cfg.n))
    np.testing.assert_allclose(fine(op, 1, X, "linear"), X @ F.T, rtol=0, atol=1e-12)
    np.testing.assert_allclose(fine(op, 1, X, "adjoint"), X @ F, rtol=0, atol=1e-12)
    assert np.linalg.norm(F - F.T) > 1e-4 * np.linalg.norm(F)
