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


class _Part:
    def __init__(self, cp, anchor, deformation, radius, thresholds):
        self.cp, self.anchor = cp, tuple(int(v) for v in anchor)
        self.deformation = tuple(float(v) for v in deformation)
        self.search_radius = int(radius)
        self.thresholds = None if thresholds is None else np.asarray(thresholds, dtype=np.float64)


class _Dec:
    """Calibrated decomposed model carrier (attribute contract of
    model.py:99-168: root_cp, parts, bias, root_thresholds, channels)."""

    def __init__(self, root_cp, parts, bias, root_thresholds):
        self.root_cp, self.parts, self.bias = root_cp, tuple(parts), float(bias)
        self.root_thresholds = (None if root_thresholds is None
                                else np.asarray(root_thresholds, dtype=np.float64))

    @property
    def channels(self):
        return self.root_cp.factors_c.shape[0]

    @property
    def calibrated(self):
        return self.root_thresholds is not None and all(p.thresholds is not None
                                                        for p in self.parts)


def golden_pruned(g, k):
    """(calibrated dec, pyramid, planted positives, tau) of detect_pruned.npz case k."""
    pre = f"q{k}"
    parts = [_Part(golden_cp(g, f"{pre}_pcp{i}"), g[f"{pre}_part{i}_anchor"],
                   g[f"{pre}_part{i}_def"], g[f"{pre}_part{i}_r"], g[f"{pre}_part{i}_thr"])
             for i in range(int(g[f"{pre}_nparts"]))]
    dec = _Dec(golden_cp(g, f"{pre}_rcp"), parts, g[f"{pre}_bias"], g[f"{pre}_root_thr"])
    pyr = [g[f"{pre}_level{i}"] for i in range(int(g[f"{pre}_nlevels"]))]
    return dec, pyr, g[f"{pre}_planted"], float(g[f"{pre}_tau"])
