"""The bound formulas against hand-evaluated values (tests/golden/bounds_tiny.txt):
eqs. error_bound_initial, error_bound_eps_delta, error_bound_eps_delta2,
error_bound_eps, error_bound_eps_inf_time, apost_bound and
apost_bound_sup, and eq. bounds_delta_eps.  A dropped
term, a wrong binomial, an off-by-one summation limit or a spurious factor
changes at least one of these numbers.  The library's host routine pr_bounds
is checked against the same golden values (it must not merely agree with the
oracle)."""
import os

import numpy as np
import pytest

from oracle import bounds
from oracle.rsvd import Truncated, delta_eps

HERE = os.path.dirname(os.path.abspath(__file__))
DELTA, EPS, N = 0.5, 0.25, 3
BNORM = np.array([1.0, 2.0, 3.0, 4.0])
E0 = np.array([0.0, 1.0, 1.0, 1.0])
UPD = np.array([0.0, 1.0, 2.0, 4.0])


def _golden():
    rows = []
    with open(os.path.join(HERE, "golden", "bounds_tiny.txt")) as f:
        for ln in f:
            ln = ln.split("#")[0].split()
            if ln:
                rows.append((ln[0], int(ln[1]), int(ln[2]), float(ln[3])))
    return rows


GOLDEN = _golden()


def _oracle(kind, n, k):
    return {
        "initial": lambda: bounds.a_priori_initial(DELTA, EPS, BNORM, n),
        "eps_delta2": lambda: bounds.a_priori_k(DELTA, EPS, BNORM, n, k),
        "eps_delta": lambda: bounds.a_priori_from_e0(DELTA, EPS, E0, n, k),
        "eps": lambda: bounds.a_priori_eps(EPS, N, k, E0),
        "eps_inf_time": lambda: bounds.a_priori_eps_inf_time(DELTA, EPS, N, k, E0),
        "apost": lambda: bounds.a_posteriori(DELTA, EPS, UPD, n),
        "apost_sup": lambda: bounds.a_posteriori_sup(DELTA, EPS, UPD),
    }[kind]()


@pytest.mark.parametrize("kind,n,k,value", GOLDEN)
def test_oracle_bound_golden(kind, n, k, value):
    assert _oracle(kind, n, k) == pytest.approx(value, rel=1e-15, abs=1e-300)


def test_pr_bounds_golden():
    """libpr's pr_bounds (host code, no GPU needed) on the golden case."""
    from paper_2508_08873_b200 import bounds as pr_bounds
    upd = UPD[None, :]
    # k = 1..3 rows of the a priori output need K = 3 update rows (only row 0 is used by apost)
    out = pr_bounds(DELTA, EPS, BNORM, np.repeat(upd, 3, axis=0))
    for kind, n, k, value in GOLDEN:
        if kind == "initial":
            assert out["apriori"][0, n] == pytest.approx(value, rel=1e-14)
        elif kind == "eps_delta2":
            assert out["apriori"][k, n] == pytest.approx(value, rel=1e-14, abs=1e-300)
        elif kind == "apost":
            assert out["apost"][0, n] == pytest.approx(value, rel=1e-14, abs=1e-300)
        elif kind == "apost_sup":
            assert out["apost_sup"][0] == pytest.approx(value, rel=1e-14)


def test_delta_eps_definition():
    """eq. bounds_delta_eps with the computed sigma_{n,R+1}:
    delta = max_n sigma_{n,1}, eps = max_n sigma_{n,k+1} -- over intervals, not
    sigma_{n,k} and not the last computed value."""
    sig = [np.array([0.9, 0.5, 0.2, 0.1]), np.array([0.95, 0.4, 0.3, 0.05]),
           np.array([0.7, 0.6, 0.25, 0.2])]
    tr = [Truncated(U=np.zeros((4, 2)), sigma=s, V=np.zeros((4, 2)), k=2) for s in sig]
    d, e = delta_eps(tr)
    assert d == 0.95 and e == 0.3
    tr1 = [Truncated(U=np.zeros((4, 1)), sigma=s, V=np.zeros((4, 1)), k=1) for s in sig]
    assert delta_eps(tr1) == (0.95, 0.6)
