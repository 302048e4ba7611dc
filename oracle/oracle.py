"""ctypes loaders for the parity checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
`--impl reference`) import this module; the product package never does.

  Oracle   libqvoracle.so     C restatement of the reference path (qv_oracle.c)
  RefEngine _ref/libqvsim_ref.so  the unmodified reference engine + ref_driver.cpp

Gate arrays use the qvg_gate layout (include/qvg.h) as a numpy structured
dtype, so the very same bytes feed the oracle, the reference and libqvg.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

GATE_DTYPE = np.dtype(
    [("kind", "<u4"), ("target", "<u4"), ("control", "<i4"), ("flags", "<u4"), ("u", "<f8", (8,))],
    align=False,
)
assert GATE_DTYPE.itemsize == 80

_P = ctypes.c_void_p
_U32, _U64, _I32, _DBL = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


def build_oracle() -> None:
    """make -C oracle (the C restatement; the reference only when present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


class Oracle:
    """The C restatement (qv_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "libqvoracle.so")
        if not os.path.exists(path):
            build_oracle()
        lib = ctypes.CDLL(path)
        lib.qvo_random_circuit.argtypes = [_U32, _U32, _U64, _P, _P]
        lib.qvo_random_circuit.restype = _U32
        lib.qvo_apply.argtypes = [_U32, _P, _P, _U64]
        lib.qvo_apply.restype = ctypes.c_int
        lib.qvo_basis_state.argtypes = [_U32, _P, _U64]
        lib.qvo_probabilities.argtypes = [_U64, _P, _P]
        lib.qvo_norm.argtypes = [_U64, _P]
        lib.qvo_norm.restype = _DBL
        lib.qvo_max_deviation.argtypes = [_U64, _P, _P]
        lib.qvo_max_deviation.restype = _DBL
        self.lib = lib

    def random_circuit(self, n: int, depth: int, seed: int):
        ops = np.zeros(depth, GATE_DTYPE)
        names = np.zeros(depth, np.int32)
        self.lib.qvo_random_circuit(n, depth, seed, _ptr(ops), _ptr(names))
        return ops, names

    def basis(self, n: int, index: int = 0) -> np.ndarray:
        amps = np.zeros(1 << n, np.complex128)
        amps[index] = 1.0
        return amps

    def apply(self, n: int, amps: np.ndarray, ops: np.ndarray) -> np.ndarray:
        """In place on a complex128 array of 2^n amplitudes."""
        assert amps.dtype == np.complex128 and amps.size == (1 << n) and amps.flags.c_contiguous
        ops = np.ascontiguousarray(ops, GATE_DTYPE)
        rc = self.lib.qvo_apply(n, _ptr(amps), _ptr(ops), len(ops))
        if rc:
            raise ValueError(f"oracle rejected op {rc - 1}")
        return amps

    def simulate(self, n: int, ops: np.ndarray, init_index: int = 0) -> np.ndarray:
        return self.apply(n, self.basis(n, init_index), ops)

    def probabilities(self, amps: np.ndarray) -> np.ndarray:
        out = np.empty(amps.size, np.float64)
        self.lib.qvo_probabilities(amps.size, _ptr(amps), _ptr(out))
        return out

    def norm(self, amps: np.ndarray) -> float:
        return self.lib.qvo_norm(amps.size, _ptr(amps))

    def max_deviation(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, np.complex128)
        b = np.ascontiguousarray(b, np.complex128)
        return self.lib.qvo_max_deviation(a.size, _ptr(a), _ptr(b))


class RefEngine:
    """The unmodified reference engine (oracle/_ref, built by `make -C oracle ref`)."""

    PATH = os.path.join(HERE, "_ref", "libqvsim_ref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        lib = ctypes.CDLL(self.PATH)
        lib.qvr_last_error.restype = ctypes.c_char_p
        lib.qvr_last_error_kind.restype = ctypes.c_char_p
        lib.qvr_random_circuit.argtypes = [_U32, _U32, _U64, _P, ctypes.c_char_p, _U64]
        lib.qvr_simulate_dense.argtypes = [_U32, _P, _U64, _P]
        lib.qvr_store_create.argtypes = [ctypes.c_char_p, _U32, _U64, _U64]
        lib.qvr_store_create.restype = _P
        lib.qvr_store_load.argtypes = [_P, _P]
        lib.qvr_store_apply.argtypes = [_P, _P, _U64, ctypes.c_char_p, _U32, _U64, ctypes.POINTER(_DBL)]
        lib.qvr_store_read.argtypes = [_P, _P]
        lib.qvr_store_norm.argtypes = [_P, ctypes.POINTER(_DBL)]
        lib.qvr_store_sync.argtypes = [_P]
        lib.qvr_store_destroy.argtypes = [_P]
        lib.qvr_store_open.argtypes = [ctypes.c_char_p]
        lib.qvr_store_open.restype = _P
        lib.qvr_store_close.argtypes = [_P]
        lib.qvr_store_path.argtypes = [_P, ctypes.c_char_p, _U64]
        lib.qvr_parse.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int, _P, _U64, ctypes.POINTER(_U64),
                                  ctypes.POINTER(_U32), ctypes.POINTER(_U64), ctypes.c_char_p, _U64]
        self.lib = lib

    def _check(self, rc: int):
        if rc:
            raise RuntimeError(self.lib.qvr_last_error().decode())

    def random_circuit(self, n: int, depth: int, seed: int):
        ops = np.zeros(depth, GATE_DTYPE)
        buf = ctypes.create_string_buffer(1 << 20)
        self._check(self.lib.qvr_random_circuit(n, depth, seed, _ptr(ops), buf, len(buf)))
        return ops, buf.value.decode()

    def parse(self, text: str, qubits: int | None = None, strict: bool = False):
        """The reference's parse_circuit: (n_qubits, ops, serialized text), or
        ("ParseError", line) / ("Error", message) when it throws."""
        cap = 4096
        ops = np.zeros(cap, GATE_DTYPE)
        count, n, line = _U64(0), _U32(0), _U64(0)
        buf = ctypes.create_string_buffer(1 << 20)
        rc = self.lib.qvr_parse(text.encode(), -1 if qubits is None else qubits, int(strict), _ptr(ops), cap,
                                ctypes.byref(count), ctypes.byref(n), ctypes.byref(line), buf, len(buf))
        if rc == 2:
            return ("ParseError", line.value)
        if rc:
            return ("Error", self.lib.qvr_last_error().decode())
        return n.value, ops[:count.value].copy(), buf.value.decode()

    def simulate_dense(self, n: int, ops: np.ndarray) -> np.ndarray:
        out = np.zeros(1 << n, np.complex128)
        ops = np.ascontiguousarray(ops, GATE_DTYPE)
        self._check(self.lib.qvr_simulate_dense(n, _ptr(ops), len(ops), _ptr(out)))
        return out

    def store(self, n: int, block_amps: int = 65536, init_index: int = 0, scratch: str | None = None):
        return RefStore(self, n, block_amps, init_index, scratch)

    def open_store(self, path: str, n: int):
        """An existing QVSV file through the reference's BlockStore::open; closing
        it keeps the file."""
        st = RefStore.__new__(RefStore)
        st.eng, st.n, st.keep = self, n, True
        st.h = self.lib.qvr_store_open(path.encode())
        if not st.h:
            raise RefError(self.lib.qvr_last_error_kind().decode(), self.lib.qvr_last_error().decode())
        return st

    def open_error(self, path: str):
        """None when the reference opens the file, else its error class name."""
        h = self.lib.qvr_store_open(path.encode())
        if h:
            self.lib.qvr_store_close(h)
            return None
        return self.lib.qvr_last_error_kind().decode()


class RefError(RuntimeError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def default_scratch() -> str:
    d = os.environ.get("QVSIM_TEST_DIR")  # reference tests/test_util.hpp:14-49
    if d:
        return d
    return "/dev/shm" if os.path.isdir("/dev/shm") and os.access("/dev/shm", os.W_OK) else "/tmp"


class RefStore:
    """A reference BlockStore with apply_circuit through a chosen strategy."""

    def __init__(self, eng: RefEngine, n: int, block_amps: int, init_index: int, scratch: str | None):
        self.eng, self.n = eng, n
        self.h = eng.lib.qvr_store_create((scratch or default_scratch()).encode(), n, block_amps, init_index)
        if not self.h:
            raise RuntimeError(eng.lib.qvr_last_error().decode())

    def load(self, amps: np.ndarray):
        amps = np.ascontiguousarray(amps, np.complex128)
        self.eng._check(self.eng.lib.qvr_store_load(self.h, _ptr(amps)))

    def apply(self, ops: np.ndarray, strategy: str = "paired-cached", workers: int = 1,
              cache_bytes: int = 64 << 20) -> float:
        ops = np.ascontiguousarray(ops, GATE_DTYPE)
        wall = _DBL(0.0)
        self.eng._check(self.eng.lib.qvr_store_apply(self.h, _ptr(ops), len(ops), strategy.encode(),
                                                     workers, cache_bytes, ctypes.byref(wall)))
        return wall.value

    def read(self) -> np.ndarray:
        out = np.zeros(1 << self.n, np.complex128)
        self.eng._check(self.eng.lib.qvr_store_read(self.h, _ptr(out)))
        return out

    def norm(self) -> float:
        v = _DBL(0.0)
        self.eng._check(self.eng.lib.qvr_store_norm(self.h, ctypes.byref(v)))
        return v.value

    def sync(self):
        self.eng._check(self.eng.lib.qvr_store_sync(self.h))

    def path(self) -> str:
        buf = ctypes.create_string_buffer(4096)
        self.eng._check(self.eng.lib.qvr_store_path(self.h, buf, len(buf)))
        return buf.value.decode()

    def amplitudes(self) -> np.ndarray:
        """Read-only memory map of the store's amplitude payload (the QVSV
        layout: a 32-byte header, then 2^n little-endian complex128,
        reference store.hpp:13-29). Call sync() first."""
        return np.memmap(self.path(), dtype=np.complex128, mode="r", offset=32, shape=(1 << self.n,))

    def close(self):
        if self.h:
            if getattr(self, "keep", False):
                self.eng.lib.qvr_store_close(self.h)
            else:
                self.eng.lib.qvr_store_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
