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


_CK = [0x9e3779b97f4a7c15, 0xc2b2ae3d27d4eb4f, 0x165667b19e3779f9, 0x27d4eb2f165667c5, 0xd6e8feb86659fd93,
       0xff51afd7ed558ccd]


def _ck_mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return z ^ (z >> np.uint64(31))


def checksums_numpy(amps, chunk_amps, base_index=0):
    """numpy restatement of the device chunk checksums (qvg_readout.cuh
    k_checksum, qvg_checksums): per chunk, two uint64 sums (mod 2^64) of
    splitmix-mixed amplitude bit patterns, salted with the global index."""
    K = [np.uint64(k) for k in _CK]
    if amps.dtype == np.complex128:
        bits = amps.view(np.uint64).reshape(-1, 2)
        re, im = bits[:, 0], bits[:, 1]
    else:
        bits = amps.view(np.uint32).reshape(-1, 2).astype(np.uint64)
        re, im = bits[:, 0], bits[:, 1]
    with np.errstate(over="ignore"):
        i = np.arange(base_index, base_index + amps.size, dtype=np.uint64)
        w0 = _ck_mix(re ^ (i * K[0])) + _ck_mix(im ^ (i * K[1] + K[2]))
        w1 = _ck_mix(re ^ (i * K[3] + K[4])) + _ck_mix(im ^ (i * K[5]))
        out = np.zeros((amps.size // chunk_amps, 2), np.uint64)
        out[:, 0] = w0.reshape(-1, chunk_amps).sum(axis=1, dtype=np.uint64)
        out[:, 1] = w1.reshape(-1, chunk_amps).sum(axis=1, dtype=np.uint64)
    return out


def algorithmic_bytes(n, amp_bytes, op):
    """SURVEY §8d's bytes of one gate pass, restated from the table (not from
    the planner): 2 * touched * S with touched = the amplitudes the gate reads
    and writes -- all of them for a dense or general-diagonal 1q gate, the
    control = 1 half for a controlled gate, the target = 1 half for
    diag(1, d), the |11> quarter for a controlled diag(1, d), nothing for the
    identity -- charged in whole 32-B sectors when the touched runs are
    shorter than a sector, and never more than the whole state."""
    u = [float(x) for x in op["u"]]
    ctl, tgt = int(op["control"]), int(op["target"])
    full = 2 * (1 << n) * amp_bytes
    diag = u[2] == 0 and u[3] == 0 and u[4] == 0 and u[5] == 0
    phase = diag and u[0] == 1 and u[1] == 0
    if phase and u[6] == 1 and u[7] == 0:
        return 0
    forced = []  # bits that must be 1 in a touched amplitude
    if ctl >= 0:
        forced.append(ctl)
    if phase:
        forced.append(tgt)
    b = full >> len(forced)
    if forced:
        run = (1 << min(forced)) * amp_bytes
        if run < 32:
            b *= 32 // run
    return min(b, full)
