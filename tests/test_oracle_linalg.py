"""Pins for oracle/linalg.py: Householder QR and one-sided Jacobi
SVD, against LAPACK (numpy.linalg) and exact special cases."""
import numpy as np
import pytest

from oracle.linalg import householder_qr, jacobi_svd


@pytest.mark.parametrize("n,l", [(50, 7), (300, 40), (12, 12)])
def test_householder_qr(n, l):
    rng = np.random.default_rng(n + l)
    Y = rng.standard_normal((n, l))
    Q, R = householder_qr(Y)
    assert np.max(np.abs(Q.T @ Q - np.eye(l))) < 1e-14
    assert np.max(np.abs(Q @ R - Y)) < 1e-14 * np.max(np.abs(Y)) * l
    Qn, Rn = np.linalg.qr(Y)
    sgn = np.sign(np.diag(R)) * np.sign(np.diag(Rn))
    np.testing.assert_allclose(Q * sgn, Qn, atol=1e-12)


def test_householder_qr_rank_deficient():
    """Numerically rank-deficient block (like the snapshot blocks, SURVEY finding 6):
    Q stays orthonormal and spans range(Y)."""
    rng = np.random.default_rng(5)
    n, l, r = 200, 12, 5
    Y = rng.standard_normal((n, r)) @ rng.standard_normal((r, l))
    Y[:, -1] *= 1e-30
    Q, R = householder_qr(Y)
    assert np.max(np.abs(Q.T @ Q - np.eye(l))) < 1e-14
    assert np.linalg.norm(Y - Q @ (Q.T @ Y)) < 1e-14 * np.linalg.norm(Y)


@pytest.mark.parametrize("shape", [(12, 12), (40, 40), (9, 5)])
def test_jacobi_svd_against_lapack(shape):
    rng = np.random.default_rng(shape[0])
    M = rng.standard_normal(shape) @ np.diag(np.logspace(0, -8, shape[1]))
    U, s, V = jacobi_svd(M)
    sref = np.linalg.svd(M, compute_uv=False)
    assert np.max(np.abs(s - sref)) < 1e-14 * sref[0]
    assert np.max(np.abs(U @ np.diag(s) @ V.T - M)) < 1e-13 * sref[0]
    assert np.max(np.abs(V.T @ V - np.eye(shape[1]))) < 1e-13
    assert np.all(np.diff(s) <= 0)
    # sign convention Z10
    for r in range(V.shape[1]):
        assert V[np.argmax(np.abs(V[:, r])), r] > 0


def test_jacobi_svd_special_cases():
    D = np.diag([3.0, -1.0, 2.0])                   # S:80-83 style: diagonal
    U, s, V = jacobi_svd(D)
    np.testing.assert_allclose(s, [3.0, 2.0, 1.0], rtol=1e-15)
    th = 0.3
    Rm = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])   # rotation
    _, s2, _ = jacobi_svd(Rm)
    np.testing.assert_allclose(s2, [1.0, 1.0], rtol=1e-15)
    L = np.tril(np.random.default_rng(1).standard_normal((16, 16)))        # M = R_Z^T shape
    _, s3, _ = jacobi_svd(L)
    np.testing.assert_allclose(s3, np.linalg.svd(L, compute_uv=False), rtol=0, atol=1e-14 * s3[0])
