"""The C-ABI library loads and exports every symbol include/pr.h declares; host
logic (pr_bounds, argument validation that returns before any launch) is
checked on the CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2508_08873_b200 import build as B
    B.build()
    from paper_2508_08873_b200 import _lib
    return _lib.lib()


def _declared():
    hdr = open(os.path.join(ROOT, "include", "pr.h")).read()
    return sorted(set(re.findall(r"\b(pr_[a-z0-9_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(L):
    from paper_2508_08873_b200 import _lib
    decl = _declared()
    assert len(decl) >= 15
    assert sorted(_lib.EXPORTS) == decl
    for name in decl:
        assert hasattr(L, name), name
    # the symbols are exported with C linkage from libpr.so itself
    out = os.popen(f"nm -D --defined-only {_lib.SO_PATH}").read()
    for name in decl:
        assert re.search(rf"\bT {name}\b", out), name


def test_so_is_sm100a(L):
    from paper_2508_08873_b200 import _lib
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.SO_PATH}").read()
    assert "sm_100a" in out


def test_validation_before_launch(L):
    from paper_2508_08873_b200 import _lib
    h = ctypes.c_void_p()
    a = np.zeros(4)
    p = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    assert L.pr_op_create_tridiag(1, p, p, p, None, None, 0.1, ctypes.byref(h)) == _lib.PR_EINVAL
    assert L.pr_op_create_tridiag(4, p, p, p, None, None, -1.0, ctypes.byref(h)) == _lib.PR_EINVAL
    assert b"dt" in L.pr_last_error()
    assert L.pr_fine_propagate(None, 0, 0, 1, 1, 1, None, None, 0, None, 0, None, 0, None) == _lib.PR_EINVAL
    assert L.pr_bounds(0.5, 0.1, 0, 1, None, None, None, None, None) == _lib.PR_EINVAL
    hs = (ctypes.c_void_p * 2)()
    assert L.pr_comm_create_local(0, hs) == _lib.PR_EINVAL
    assert L.pr_comm_info(None, None, None) == _lib.PR_EINVAL
    assert L.pr_comm_create_nccl(2, 2, None, ctypes.byref(h)) == _lib.PR_EINVAL
    assert L.pr_build_coarse(None, 4, 0, 4, 1, 1, 0, 0, None, None, None, ctypes.byref(h)) == _lib.PR_EINVAL


def test_pr_bounds_matches_oracle_formulas(L):
    from oracle import bounds as OB
    from paper_2508_08873_b200.api import bounds
    rng = np.random.default_rng(0)
    N, K = 12, 5
    bnorm = rng.uniform(0.1, 2.0, N + 1)
    upd = rng.uniform(0, 1e-3, (K, N + 1)) * (0.1 ** np.arange(K))[:, None]
    upd[:, 0] = 0
    for delta, eps in ((0.9, 0.05), (1.0, 0.2), (0.3, 1e-6)):
        r = bounds(delta, eps, bnorm, upd)
        for k in range(K + 1):
            for n in range(N + 1):
                ref = OB.a_priori_k(delta, eps, bnorm, n, k)
                assert abs(r["apriori"][k, n] - ref) <= 1e-12 * max(ref, 1e-300)
        for k in range(1, K + 1):
            for n in range(N + 1):
                ref = OB.a_posteriori(delta, eps, upd[k - 1], n)
                assert abs(r["apost"][k - 1, n] - ref) <= 1e-13 * max(ref, 1e-300)
            if delta < 1:
                ref = OB.a_posteriori_sup(delta, eps, upd[k - 1])
                assert abs(r["apost_sup"][k - 1] - ref) <= 1e-13 * ref
            else:
                assert np.isnan(r["apost_sup"][k - 1])
