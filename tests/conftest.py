import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full-size parity)")


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()


@pytest.fixture(autouse=True)
def _fhwt_tuning(monkeypatch):
    """The library honours its FHWT_* sweep knobs only with FHWT_TUNING=1; the
    A/B tests below set knobs through monkeypatch, so the gate is open for every test (the test of
    the gate itself removes it)."""
    monkeypatch.setenv("FHWT_TUNING", "1")
