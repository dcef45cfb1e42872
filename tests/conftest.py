import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"
GOLDEN_CASES = ["sphere2_default", "sphere3_l32_eta2_o4", "config1_sphere4",
                "torus_32_16_4_default", "prism_20_40_2_default"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libh2b.so")


_cache = {}


def load_golden(name):
    if name not in _cache:
        from paper_1811_05731_b200.io import load_npz
        _cache[name] = load_npz(GOLDEN / f"{name}.npz")
    return _cache[name]


@pytest.fixture(params=GOLDEN_CASES)
def golden(request):
    op, ex = load_golden(request.param)
    return request.param, op, ex


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
