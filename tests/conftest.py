"""Shared fixtures. Markers: ``gpu`` = needs a CUDA device (run on the B200 box)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

# Table 3 two-layer set: soft layer over a stiff half-space
TWO_LAYER = [(1600.0, 400.0, 1850.0), (5800.0, 3000.0, 2700.0)]
STIFF = [(5800.0, 3000.0, 2700.0)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def lame(table):
    lam = np.array([rho * (vp * vp - 2 * vs * vs) for vp, vs, rho in table])
    mu = np.array([rho * vs * vs for vp, vs, rho in table])
    return lam, mu


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def reference():
    from oracle import Oracle, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref/libtsref.so not built (reference sources absent)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def checker():
    """The checker for the CUDA path: the reference itself when built, else the pinned C port."""
    from oracle import Oracle, have_reference
    return Oracle("reference" if have_reference() else "port")
