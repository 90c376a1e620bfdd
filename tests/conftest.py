"""Shared fixtures. `-m gpu` tests need a B200; everything else runs on CPU."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    """ctypes handle on oracle/liboracle.so (the CPU checker; built on demand)."""
    so = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")],
                       check=True, capture_output=True)
    from tests import oracle_py
    return oracle_py.Oracle(ctypes.CDLL(so))


@pytest.fixture(scope="session")
def golden_configs():
    return load_golden("configs.npz")


@pytest.fixture(scope="session")
def golden_conv():
    return load_golden("conv_cases.npz")


@pytest.fixture(scope="session")
def golden_kats():
    return load_golden("kats.npz")


@pytest.fixture(scope="session")
def golden_appendix():
    return load_golden("appendix_a.npz")
