"""A priori and a posteriori error bounds -- TEST INFRASTRUCTURE ONLY.

Theorem general_convergence (eqs. error_bound_initial,
error_bound_eps_delta, error_bound_eps_delta2, error_bound_eps,
error_bound_eps_inf_time) and the a posteriori theorem
(P:599-612), written out term by term.  delta, eps as in eq. bounds_delta_eps
(P:407-411); norms are Euclidean.  Index conventions follow the
paper: n = 1..N, m the summation index, b_0 := u_0.
"""
from __future__ import annotations

from math import comb

import numpy as np


def a_priori_initial(delta, eps, bnorm, n):
    """eq. error_bound_initial: sum_{m=0}^{n-1} min(2 delta, (n-m) eps) delta^{n-m-1} ||b_m||."""
    return sum(min(2 * delta, (n - m) * eps) * delta ** (n - m - 1) * bnorm[m] for m in range(n))


def a_priori_k(delta, eps, bnorm, n, k):
    """eq. error_bound_eps_delta2: 2 eps^k sum_{m=0}^{n-k-1} C(n-m, k) delta^{n-m-k} ||b_m||."""
    if k == 0:
        return a_priori_initial(delta, eps, bnorm, n)
    return 2 * eps ** k * sum(comb(n - m, k) * delta ** (n - m - k) * bnorm[m]
                              for m in range(0, n - k))


def a_priori_from_e0(delta, eps, e0, n, k):
    """eq. error_bound_eps_delta: eps^k sum_{m=1}^{n-k} C(n-m, k-1) delta^{n-m-k} ||e^0_m||."""
    return eps ** k * sum(comb(n - m, k - 1) * delta ** (n - m - k) * e0[m]
                          for m in range(1, n - k + 1))


def a_posteriori(delta, eps, upd_k, n):
    """eq. apost_bound: eps sum_{m=1}^{n-1} delta^{n-m-1} ||u^k_m - u^{k-1}_m||."""
    return eps * sum(delta ** (n - m - 1) * upd_k[m] for m in range(1, n))


def a_posteriori_sup(delta, eps, upd_k):
    """eq. apost_bound_sup (delta < 1): eps/(1-delta) max_n ||u^k_n - u^{k-1}_n||."""
    assert delta < 1
    return eps / (1 - delta) * float(np.max(upd_k[1:]))


def spectral_contraction(sigma_next, e0max, k):
    """Corollary spectral_bound: sigma_{R+1}^k max_{n<=N-k} ||e^0_n||."""
    return sigma_next ** k * e0max


def a_priori_eps(eps, N, k, e0):
    """eq. error_bound_eps (delta <= 1): max_n ||e^k_n|| <= C(N, k) eps^k max_{1<=m<=N-k} ||e^0_m||."""
    if N - k < 1:
        return 0.0
    return comb(N, k) * eps ** k * max(e0[m] for m in range(1, N - k + 1))


def a_priori_eps_inf_time(delta, eps, N, k, e0):
    """eq. error_bound_eps_inf_time (delta < 1):
    max_n ||e^k_n|| <= (eps / (1 - delta))^k max_{1<=n<=N-k} ||e^0_n||."""
    assert delta < 1
    if N - k < 1:
        return 0.0
    return (eps / (1.0 - delta)) ** k * max(e0[n] for n in range(1, N - k + 1))


def efficiency(delta, eps, upd_k, traj_err_k, N):
    """eq. def_efficiency, as printed (the max over 1 <= n < N,
    reading Z21):
        eta^k = max_t ||u^k(t) - u(t)|| / max_{1<=n<N} eps sum_{m=1}^{n-1} delta^{n-m-1} ||u^k_m - u^{k-1}_m||."""
    den = max(a_posteriori(delta, eps, upd_k, n) for n in range(1, N))
    return traj_err_k / den
