"""Pins of the oracle's time-dependent pencil fine solver (SURVEY 8(f) rows
1-2; the paper's Experiment 2, eq. ex2) to things other than
itself: the dense product of the step matrices (numpy.linalg.solve, brute
force), the Euclidean transpose of that product (reverse step order, R-ADJ),
the undamped constant mode of the Neumann problem (A(t) 1 = 0 => F' 1 = 1,
P:511-513), the exact load-vector integral, and affinity
F v = F' v + F 0 (eq. F_n_affine)."""
import numpy as np
import pytest

from oracle.fine import OpPencil, dense_step_product, fine, make_op
from oracle.rsvd import rsvd_interval
from workloads import exp2
from workloads import generators as G
from workloads.configs import get

pytestmark = pytest.mark.filterwarnings("ignore")


@pytest.mark.parametrize("name", ["E2", "E2FD"])
@pytest.mark.parametrize("interval", [1, 6, 10])
def test_pencil_linear_and_adjoint_match_dense_step_product(name, interval):
    cfg = get(name)
    op = make_op(cfg)
    F = dense_step_product(op, interval)
    E = np.eye(cfg.n)
    Fl = fine(op, interval, E, "linear").T          # columns F' e_j
    Fa = fine(op, interval, E, "adjoint").T         # columns F'^T e_j
    s = np.linalg.norm(F, 2)
    assert np.linalg.norm(Fl - F, 2) <= 1e-12 * s
    assert np.linalg.norm(Fa - F.T, 2) <= 1e-12 * s


def test_pencil_adjoint_order_is_reversed():
    """The steps differ (kappa depends on t), so the adjoint in forward step
    order is a different (wrong) operator: the pin separates the two."""
    cfg = get("E2FD")
    op = make_op(cfg)
    F = dense_step_product(op, 3)
    wrong = np.eye(cfg.n)
    for j in range(1, op.m + 1):                     # transposed steps, FORWARD order
        g = 2 * op.m + j
        a, d, c = (arr[g - 1] for arr in op.L)
        Lg = np.diag(d) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
        wrong = np.linalg.solve(Lg.T, wrong)
    assert np.linalg.norm(wrong - F.T, 2) > 1e-6 * np.linalg.norm(F, 2)
    assert not np.allclose(F @ F.T, F.T @ F, atol=1e-6)     # F' is not normal


@pytest.mark.parametrize("name", ["E2", "E2FD"])
def test_pencil_constant_mode_is_undamped(name):
    cfg = get(name)
    op = make_op(cfg)
    one = np.ones((1, cfg.n))
    for q in (1, 4, 10):
        y = fine(op, q, one, "linear")
        assert np.max(np.abs(y - 1.0)) < 1e-13
    # hence sigma_1 >= 1 for every interval (delta = 1 in P:511-513)
    t = rsvd_interval(op, 2, cfg.k, cfg.p, cfg.seed_omega)
    assert t.sigma[0] >= 1.0 - 1e-13


def test_exp2_load_vector_integrates_exactly():
    """sum_i int f phi_i dx = int (1 + cos 3 pi x) dx = 1 (partition of unity);
    and the hat-function integrals against quadrature."""
    from scipy.integrate import quad
    for n in (11, 101):
        b = exp2.load_space("exp2_fem", n)
        assert abs(b.sum() - 1.0) < 1e-14
        h = 1.0 / (n - 1)
        x = exp2.nodes(n)
        for i in (0, 1, n // 2, n - 1):
            phi = lambda t: max(0.0, 1.0 - abs(t - x[i]) / h)
            ref = quad(lambda t: (1.0 + np.cos(3 * np.pi * t)) * phi(t), max(0, x[i] - h),
                       min(1, x[i] + h), epsabs=1e-15)[0]
            assert abs(b[i] - ref) < 1e-13


def test_exp2_stiffness_rows_sum_to_zero_and_mass_rows():
    for n in (11, 101):
        a, d, c = exp2.stiffness(n, 0.37)
        assert np.max(np.abs(a + d + c)) < 1e-12 * np.max(np.abs(d))
        ms, md, mp, rows = exp2.mass(n)
        assert np.allclose(ms + md + mp, rows, rtol=0, atol=1e-16)
        assert abs(rows.sum() - 1.0) < 1e-14            # int 1 dx


@pytest.mark.parametrize("name", ["E2", "E2FD"])
def test_pencil_affine_is_affine(name):
    cfg = get(name)
    op = make_op(cfg)
    src = G.source_1d(cfg)
    rng = np.random.default_rng(3)
    v = rng.standard_normal((2, cfg.n))
    for q in (1, 7):
        Fv = fine(op, q, v, "affine", src)
        F0 = fine(op, q, np.zeros((1, cfg.n)), "affine", src)
        Flv = fine(op, q, v, "linear")
        assert np.linalg.norm(Fv - Flv - F0) <= 1e-12 * np.linalg.norm(Fv)


def test_pencil_affine_one_step_dense():
    """One step by a dense solve of (M + dt A(t_g)) u = M u_prev + dt l(t_g)."""
    cfg = get("E2")
    (sub, diag, sup), rs, M = exp2.step_matrices("exp2_fem", cfg.n, cfg.T, cfg.N * cfg.m)
    op = OpPencil((sub, diag, sup), cfg.dt, 1, rowsum=rs, M=M)
    space, time, amp = exp2.source("exp2_fem", cfg.n, cfg.T, cfg.N * cfg.m)
    u = exp2.initial_value(cfg.n)
    g = 37
    Md = np.diag(M[1]) + np.diag(M[0][1:], -1) + np.diag(M[2][:-1], 1)
    Lg = np.diag(diag[g - 1]) + np.diag(sub[g - 1][1:], -1) + np.diag(sup[g - 1][:-1], 1)
    ref = np.linalg.solve(Lg, Md @ u + cfg.dt * time[0, g - 1] * space[0])
    got = fine(op, g, u[None, :], "affine", (space, time, amp))[0]
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
