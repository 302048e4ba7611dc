"""Shared fixtures. `-m gpu` tests need a CUDA device and the in-tree native
build; `-m "not gpu"` tests run on CPU (oracle pins, host logic, C-ABI exports)."""
import os
import sys

import numpy as np
import pytest

try:
    # torch first: once libqvg.so has mapped libcudart, `import torch` preloads
    # every CUDA wheel library, and on a host without a driver one of those
    # crashes the process (the GPU box is unaffected). Tests import torch lazily.
    import torch  # noqa: F401
except Exception:  # pragma: no cover
    pass

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libqvg.so")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def qv():
    import paper_2508_15545_b200 as qv

    return qv


def gate_array(circuit):
    """Circuit -> numpy qvg_gate records (the exact bytes libqvg consumes)."""
    from oracle.oracle import GATE_DTYPE

    return np.frombuffer(circuit.gates().tobytes(), dtype=GATE_DTYPE).copy()
