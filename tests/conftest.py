"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oplists():
    return load_json("oplists.json")


@pytest.fixture(scope="session")
def runtime_golden():
    return load_json("runtime.json")


@pytest.fixture(scope="session")
def numeric_golden():
    return np.load(os.path.join(GOLDEN, "numeric.npz"))


def divisors(p):
    return [d for d in range(1, p + 1) if p % d == 0]


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
