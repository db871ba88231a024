import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture
def pr_env(monkeypatch):
    """Set / clear PR_* diagnostic switches for one test; libpr re-reads them
    (pr_reload_env) on every change and again after the test restores them."""
    def reload():
        from paper_2508_08873_b200 import lib
        lib().pr_reload_env()

    def set_(**kv):
        for k, v in kv.items():
            if v is None:
                monkeypatch.delenv(k, raising=False)
            else:
                monkeypatch.setenv(k, str(v))
        reload()
    yield set_
    monkeypatch.undo()
    reload()
