import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtoepcuda.so")
    config.addinivalue_line("markers", "slow: long-running (large BASELINE configurations)")


def golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name}.npz not generated")
    return np.load(path)


def rel_err(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    d = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / d) if d else float(np.linalg.norm(got))


def random_complex(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
