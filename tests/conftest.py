import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhos_b200.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def max_rel_dev(a, b, floor=1e-12):
    """Per-point relative deviation (tests/conftest.py:4-9 of the reference)."""
    a = np.asarray(a)
    b = np.asarray(b)
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / denom)) if a.size else 0.0


def north_star(got, ref):
    """max|got-ref| / max|ref| (BASELINE.json north-star parity metric)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    if ref.size == 0:
        return 0.0
    s = float(np.max(np.abs(ref)))
    return float(np.max(np.abs(got - ref)) / s) if s else float(np.max(np.abs(got - ref)))


#: parity bars of BASELINE.json north_star
TOL_FP32 = 1e-5
TOL_FP64 = 1e-11


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.ensure_built()
    return torch.device("cuda", 0)
