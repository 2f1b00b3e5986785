import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


class CP:
    """Plain CP model carrier (attribute contract of decomposition.py:45-94)."""

    def __init__(self, w, a, b, c):
        self.weights = np.asarray(w, dtype=np.float64)
        self.factors_a = np.asarray(a, dtype=np.float64)
        self.factors_b = np.asarray(b, dtype=np.float64)
        self.factors_c = np.asarray(c, dtype=np.float64)

    @property
    def rank(self):
        return self.weights.size

    @property
    def dims(self):
        return (self.factors_a.shape[0], self.factors_b.shape[0], self.factors_c.shape[0])


def golden_cp(g, prefix):
    return CP(g[f"{prefix}_w"], g[f"{prefix}_a"], g[f"{prefix}_b"], g[f"{prefix}_c"])


@pytest.fixture(scope="session")
def oracle():
    from oracle import dpm_oracle

    return dpm_oracle
