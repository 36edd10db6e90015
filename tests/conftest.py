import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def unhex(v):
    if isinstance(v, str):
        return float.fromhex(v)
    return np.array([float.fromhex(s) for s in v], dtype=np.float64)


def load_golden(name):
    path = os.path.join(GOLDEN, name + ".json")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated (python oracle/make_golden.py)")
    with open(path) as f:
        return json.load(f)


def bits_equal(a, b):
    """Bitwise equality treating +0 and -0 as equal (sign of an exact zero is
    not observable through any later operation of the path)."""
    a = np.asarray(a, dtype=np.float64).copy()
    b = np.asarray(b, dtype=np.float64).copy()
    if a.shape != b.shape:
        return False
    a[a == 0] = 0.0
    b[b == 0] = 0.0
    return np.array_equal(a.view(np.int64), b.view(np.int64))


def first_mismatch(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    bad = np.nonzero(~((a == b) | (np.isnan(a) & np.isnan(b))))[0]
    if bad.size == 0:
        return None
    k = bad[0]
    return f"{bad.size} mismatches; first at {k}: {a[k]!r} vs {b[k]!r}"


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    return True
