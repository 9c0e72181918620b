import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device and the built libspa_b200.so")
    config.addinivalue_line("markers", "slow: long statistical test")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def gold_loglik():
    return golden("loglik_prior.npz")


@pytest.fixture(scope="session")
def gold_reweight():
    return golden("reweight.npz")


@pytest.fixture(scope="session")
def gold_resample():
    return golden("resample.npz")


@pytest.fixture(scope="session")
def gold_philox():
    return golden("philox.npz")


@pytest.fixture(scope="session")
def single_marker_data():
    """n=50 single-column dataset (reference tests/conftest.py:19-28)."""
    from scipy.special import expit

    from paper_1106_0322_b200.data import Dataset, standardize

    rng = np.random.default_rng(71)
    raw = rng.integers(0, 3, size=(50, 1)).astype(float)
    X = standardize(raw)
    y = (np.random.default_rng(72).random(50) < expit(X @ np.array([0.8]))).astype(float)
    return Dataset(X, y, ["snp_001"])


@pytest.fixture(scope="session")
def small_data():
    from paper_1106_0322_b200.data import named_spec, simulate_dataset

    return simulate_dataset(named_spec("a_small"))[0]
