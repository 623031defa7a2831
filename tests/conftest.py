"""Shared fixtures: golden vectors produced by the reference (tests/golden/make_golden.py)."""

import os
import sys

import numpy as np
import pytest
from scipy import sparse

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


class _Slack:
    def __init__(self, v_s):
        self.v_s = complex(v_s)


class _Zip:
    is_constant_power = True


class _Adm:
    def __init__(self, y_dd):
        self.y_dd = y_dd


class FixtureModel:
    """The hot-path model contract (y_dd, source_injection, slack, zip) of a golden file."""

    def __init__(self, d):
        shape = tuple(int(x) for x in d["ydd_shape"])
        self.admittance = _Adm(sparse.csc_matrix((d["ydd_data"], d["ydd_indices"], d["ydd_indptr"]),
                                                 shape=shape))
        self._src = np.asarray(d["src"], dtype=complex)
        self.slack = _Slack(complex(d["v_s"]))
        self.zip = _Zip()

    @property
    def n_demand(self):
        return self.admittance.y_dd.shape[0]

    def source_injection(self):
        return self._src.copy()


class Golden:
    def __init__(self, name):
        self.name = name
        self.d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        self.model = FixtureModel(self.d)
        self.S = self.d["S"]

    def __getitem__(self, k):
        return self.d[k]

    def __contains__(self, k):
        return k in self.d

    @property
    def args(self):
        m = self.model
        return m.admittance.y_dd, m.source_injection(), m.slack.v_s

    def opts(self):
        from paper_2403_04578_b200 import SolveOptions
        return SolveOptions(tolerance=float(self.d["tol"]), max_iterations=int(self.d["max_iter"]),
                            residual_tolerance=float(self.d["residual_tol"]))


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]
    return get


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
