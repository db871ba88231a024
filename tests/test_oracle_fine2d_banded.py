"""Oracle A (banded Cholesky, no sine basis) for the 2D fine solver, and the
cross-validation of oracle B (the x-sine-transform + Thomas-lines solver the
2D parity tests use) against it -- SURVEY.md §8(c) items 2 and 8.

Oracle A is pinned by itself being a direct solve of the 5-point system:
the residual of (I + dt A) x = b with A applied by its stencil (not by the
factor), and dense (I + dt A)^{-m} on a tiny grid.  Oracle B must then agree
with it on real C3 and C5 intervals to 1e-12 normwise (backward Euler,
P:648-650; eq. F_n_affine, with the moving-bump source).
"""
import functools

import numpy as np
import pytest

from oracle._clib import band_factor, band_solve
from oracle.fine import Op2DBanded, fine_2d, fine_2d_banded, make_op
from workloads import generators as G
from workloads.configs import C3, C5


def _apply_I_plus_dtA(n, dt, x):
    """(I + dt A) x for the 5-point Dirichlet Laplacian, by its stencil."""
    h2 = (1.0 / (n + 1)) ** 2
    u = np.zeros((n + 2, n + 2))
    u[1:-1, 1:-1] = x.reshape(n, n)
    lap = (4 * u[1:-1, 1:-1] - u[:-2, 1:-1] - u[2:, 1:-1] - u[1:-1, :-2] - u[1:-1, 2:]) / h2
    return (x.reshape(n, n) + dt * lap).ravel()


@pytest.mark.parametrize("n,dt", [(5, 0.3), (64, 2.0 ** -10), (255, 2.0 ** -14)])
def test_band_solve_manufactured(n, dt):
    L = band_factor(n, dt)
    b = np.random.default_rng(n).standard_normal((2, n * n))
    x = band_solve(n, L, b.copy())
    for v in range(2):
        r = _apply_I_plus_dtA(n, dt, x[v]) - b[v]
        assert np.linalg.norm(r) <= 1e-13 * np.linalg.norm(b[v])


def test_banded_fine_matches_dense_power():
    n, dt, m = 7, 0.05, 6
    h2 = (1.0 / (n + 1)) ** 2
    T = (np.diag(np.full(n, 2.0)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)) / h2
    A = np.kron(T, np.eye(n)) + np.kron(np.eye(n), T)
    F = np.linalg.matrix_power(np.linalg.inv(np.eye(n * n) + dt * A), m)
    X = np.random.default_rng(3).standard_normal((3, n, n))
    got = fine_2d_banded(Op2DBanded(n, dt, m), 1, X).reshape(3, -1)
    ref = X.reshape(3, -1) @ F.T
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


@functools.lru_cache(maxsize=None)
def _banded(name):
    cfg = {"C3": C3, "C5": C5}[name]
    return Op2DBanded(cfg.n, cfg.dt, cfg.m)


def _cross_validate(cfg, interval):
    """F_n on [probe, 0] (so F_n' probe = F(probe) - F(0) and b_n = F(0) are
    both covered) by oracle B and oracle A."""
    src = G.source_2d(cfg)
    X = np.zeros((2, cfg.n, cfg.n))
    X[0] = np.random.default_rng(interval).standard_normal((cfg.n, cfg.n))
    a = fine_2d_banded(_banded(cfg.name), interval, X, "affine", src)
    b = fine_2d(make_op(cfg), interval, X, "affine", src)
    for v in range(2):
        assert np.linalg.norm(a[v] - b[v]) <= 1e-12 * np.linalg.norm(a[v]), (interval, v)
    lin_a, lin_b = a[0] - a[1], b[0] - b[1]
    assert np.linalg.norm(lin_a - lin_b) <= 1e-12 * np.linalg.norm(X[0])


@pytest.mark.slow
@pytest.mark.parametrize("interval", [1, 64])
def test_sine_oracle_matches_banded_oracle_c3(interval):
    _cross_validate(C3, interval)


@pytest.mark.slow
def test_sine_oracle_matches_banded_oracle_c5_sampled_interval():
    _cross_validate(C5, 301)
