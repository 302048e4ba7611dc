"""B200-native gate application for the QVecOpt state-vector simulator
(arXiv 2508.15545).

The Python face mirrors the reference's ``qvsim`` package
(reference proj/python/qvsim/__init__.py:8-38): the same circuit API
(``parse_circuit``, ``random_circuit``, ``serialize_circuit`` ...) and
``apply_circuit(state, circuit, strategy=...)``, with the state held in HBM by
``StateVector`` and ``strategy="gpu"`` running the sm_100a kernels in
``libqvg.so`` (C-ABI: include/qvg.h).

There is no CPU fallback: importing this package requires the in-tree native
libraries built by ``__graft_entry__.build()`` (``make -C paper_2508_15545_b200``),
and every state operation requires a CUDA device.
"""
from __future__ import annotations

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _core  # noqa: F401  (links libqvg.so via $ORIGIN rpath)
except ImportError as exc:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_2508_15545_b200 native extension is missing or failed to load "
        f"({exc}); build it with `make -C {_HERE}` or __graft_entry__.build()"
    ) from exc

# Every public name of the native module (circuit builders, StateVector /
# StateStore, apply_circuit*, error classes, OPT_* option keys, planner and
# schedule queries) is re-exported as is.
globals().update({k: getattr(_core, k) for k in dir(_core) if not k.startswith("_")})

LIBQVG = _os.path.join(_HERE, "libqvg.so")

__all__ = sorted([k for k in dir(_core) if not k.startswith("_")] + ["LIBQVG"])

__version__ = "0.2.0"
