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

from ._core import (  # noqa: E402
    OPT_CARRIERS,
    OPT_FUSE,
    OPT_LOW_KERNEL,
    OPT_MIN_RUN,
    OPT_PRED_STORE,
    OPT_SUB_BITS,
    OPT_FMA,
    OPT_TIMING,
    OPT_EXCHANGE,
    OPT_PREFETCH,
    OPT_BATCH_EXCHANGE,
    OPT_STAGE,
    OPT_GRAPH,
    OPT_REORDER,
    OPT_CLASSES,
    OPT_TILE_QUBITS,
    QVG_ABI_VERSION,
    CapacityError,
    Circuit,
    FormatError,
    IoError,
    ParseError,
    QvsimError,
    DEFAULT_BLOCK_AMPS,
    StateStore,
    StateVector,
    ValidationError,
    top_amplitudes,
    verify_equivalence,
    apply_circuit,
    apply_circuit_host,
    circuit_from_gates,
    grid_circuit,
    haar_sweep_circuit,
    make_benchmark_circuit,
    make_gate,
    nccl_unique_id,
    parse_circuit,
    plan_passes,
    qft_circuit,
    random_circuit,
    serialize_circuit,
    shard_schedule,
    strategy_tags,
    u3_ladder_circuit,
)

LIBQVG = _os.path.join(_HERE, "libqvg.so")

__all__ = [
    "CapacityError",
    "Circuit",
    "FormatError",
    "IoError",
    "LIBQVG",
    "OPT_CARRIERS",
    "OPT_FUSE",
    "OPT_LOW_KERNEL",
    "OPT_TILE_QUBITS",
    "ParseError",
    "QVG_ABI_VERSION",
    "QvsimError",
    "StateVector",
    "ValidationError",
    "apply_circuit",
    "circuit_from_gates",
    "grid_circuit",
    "haar_sweep_circuit",
    "make_benchmark_circuit",
    "make_gate",
    "nccl_unique_id",
    "parse_circuit",
    "plan_passes",
    "qft_circuit",
    "random_circuit",
    "serialize_circuit",
    "shard_schedule",
    "strategy_tags",
    "u3_ladder_circuit",
]

__version__ = "0.1.0"
