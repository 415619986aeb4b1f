import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU-side checks")


def golden_path(name: str) -> str:
    return os.path.join(GOLDEN, f"{name}.npz")


ENGINE_CASES = [
    "uniform_off", "uniform_on", "texture_on", "texture_on_1pkt", "noise_hot_on",
    "variant_on", "noblur_on", "gain_off", "tiny_on", "odd_on",
]


@pytest.fixture(params=ENGINE_CASES)
def golden_case(request):
    import numpy as np
    return request.param, dict(np.load(golden_path(request.param), allow_pickle=False))
