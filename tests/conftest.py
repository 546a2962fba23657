import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def rng():
    # same seed as the reference's test fixture (tests/conftest.py:31-33)
    return np.random.default_rng(20240817)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_cases(name, sep="__"):
    g = load_golden(name)
    cases = {}
    for k in g.files:
        c, field = k.split(sep, 1)
        cases.setdefault(c, {})[field] = g[k]
    return [cases[c] for c in sorted(cases, key=lambda s: int(s[1:]))]


def cavitated(u, rel=1e-12):
    """Cavitated (p = 0) nodes, robust to the ~1e-19 residue the reference's
    normal-equations corner solve leaves on pinned corner nodes."""
    u = np.asarray(u)
    return u <= rel * max(1.0, float(np.max(np.abs(u))))
