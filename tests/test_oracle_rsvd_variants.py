"""The rSVD variants of §2.1 (P:301-320 power iterations; P:335-337 the
adjoint on an independent random set) in the oracle, pinned to dense SVDs of
operators with a prescribed spectrum and to the closed-form heat spectrum --
not to the formulas themselves."""
import numpy as np
import pytest

from oracle.fine import DenseOp, make_op
from oracle.rsvd import rsvd_interval
from workloads.configs import C1


def _dense(n, sig, seed=0):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return U @ np.diag(sig) @ V.T


@pytest.mark.parametrize("q,indep", [(1, False), (2, False), (0, True), (1, True)])
def test_variants_exact_when_the_sketch_spans_everything(q, indep):
    """l = n: W and V span R^n, so the computed SVD is the SVD of F'
    (non-normal operator, geometric spectrum)."""
    n = 24
    sig = 0.8 ** np.arange(n)
    F = _dense(n, sig)
    tr = rsvd_interval(DenseOp(F), 1, n, 0, 7, power_iterations=q, independent_adjoint=indep)
    np.testing.assert_allclose(tr.sigma, sig, rtol=0, atol=1e-12 * sig[0])
    X = np.random.default_rng(1).standard_normal((4, n))
    np.testing.assert_allclose(tr.apply_linear(X), X @ F.T, rtol=0, atol=1e-11)


def test_power_iterations_sharpen_a_slowly_decaying_spectrum():
    """sigma_j = 1/j: with q = 1 the leading singular values and the range
    approximation error ||(I - W W^T) F'|| improve on q = 0 (Halko et al.;
    P:312-320), and computed values never exceed the true ones (interlacing)."""
    n, k, p = 300, 6, 2
    sig = 1.0 / np.arange(1, n + 1)
    F = _dense(n, sig, seed=3)
    errs, rng_errs = [], []
    for q in (0, 1, 2):
        tr = rsvd_interval(DenseOp(F), 1, k, p, 11, power_iterations=q)
        assert np.all(tr.sigma[:k + p] <= sig[:k + p] * (1 + 1e-12))
        errs.append(np.max(np.abs(tr.sigma[:k] - sig[:k]) / sig[0]))
        G = tr.U @ np.diag(tr.sigma[:k]) @ tr.V.T
        rng_errs.append(np.linalg.norm(F - G, 2))
    assert errs[1] < 0.5 * errs[0] and errs[2] < errs[1]
    assert rng_errs[1] < rng_errs[0] and rng_errs[2] <= rng_errs[1] * (1 + 1e-9)
    assert rng_errs[2] < 1.5 * sig[k]                  # near the optimum sigma_{k+1}


def test_independent_adjoint_on_heat_matches_closed_form():
    """C1 (rank 8 numerically, l = 12): the two-sided sketch still recovers
    sigma_j = (1 + dt lam_j)^(-m) (Exp 1's Fourier argument)."""
    cfg = C1
    tr = rsvd_interval(make_op(cfg), 3, cfg.k, cfg.p, cfg.seed_omega, independent_adjoint=True)
    h = cfg.h
    lam = 4.0 / h ** 2 * np.sin(np.arange(1, cfg.n + 1) * np.pi * h / 2) ** 2
    exact = np.sort((1.0 + cfg.dt * lam) ** (-cfg.m))[::-1]
    np.testing.assert_allclose(tr.sigma[:cfg.k], exact[:cfg.k], rtol=0, atol=1e-12 * exact[0])


def test_coarse_error_estimate_brackets_the_true_error():
    """Halko-Martinsson-Tropp Lemma 4.1 estimator (adaptive p):
    the true ||F' - G'|| (dense F', tiny grid) lies below the estimate (r = 10,
    failure probability 1e-10), and the estimate is below 10 sqrt(2/pi) times
    the true norm times the largest probe norm (Cauchy-Schwarz)."""
    import numpy as np
    from oracle.fine import make_op
    from oracle.rng import gaussian_sketch
    from oracle.rsvd import coarse_error_estimate, dense_transfer, rsvd_interval
    from workloads.configs import get
    cfg = get("T1")
    op = make_op(cfg)
    for q in (1, 4):
        F = dense_transfer(op, q)
        for k, p in ((2, 1), (3, 2)):
            t = rsvd_interval(op, q, k, p, cfg.seed_omega)
            G = t.U @ np.diag(t.sigma[:k]) @ t.V.T
            true = np.linalg.norm(F - G, 2)
            est = coarse_error_estimate(op, t, q, 10, cfg.seed_omega)
            om = gaussian_sketch(cfg.seed_omega, q - 1, cfg.n, 10, stream=3)
            assert true <= est <= 10 * np.sqrt(2 / np.pi) * true * np.max(np.linalg.norm(om, axis=0)) * (1 + 1e-12)
