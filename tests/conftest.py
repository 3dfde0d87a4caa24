"""Shared fixtures.  `gpu` marks tests that need a CUDA device (run with
`-m gpu` on the B200 box); everything else runs on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "reference: needs /root/reference (absent on the GPU box)")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    have_gpu = _cuda_ok()
    have_ref = os.path.isdir(REFERENCE_SRC)
    for item in items:
        if "gpu" in item.keywords and not have_gpu:
            item.add_marker(pytest.mark.skip(reason="no CUDA device in this container"))
        if "reference" in item.keywords and not have_ref:
            item.add_marker(pytest.mark.skip(reason="/root/reference is not mounted here"))


@pytest.fixture(scope="session")
def diffpaint():
    """The live reference package (only where /root/reference is mounted)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("/root/reference is not mounted here")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import diffpaint as dp
    return dp


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
