"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything
else runs on a CPU-only host (``pytest -m "not gpu"``)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def golden_kernels():
    return load_json("kernels.json"), load_npz("kernels.npz")


@pytest.fixture(scope="session")
def golden_merge():
    return load_json("merge.json"), load_npz("merge.npz")


@pytest.fixture(scope="session")
def golden_schedules():
    return load_json("schedules.json")


@pytest.fixture(scope="session")
def golden_execute():
    return load_json("execute.json"), load_npz("execute.npz")
