import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        index = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return index, arrays


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


@pytest.fixture
def example_field():
    """The paper's 2x4 worked example (reference tests/conftest.py:15-20)."""
    return np.array([[1.2, 1.5, -2.3, -2.5], [2.5, -1.0, 2.0, 1.7]], dtype=np.float32)
