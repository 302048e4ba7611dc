"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
engine (oracle/_ref/libqvsim_ref.so, built from /root/reference by
`make -C oracle ref`). Run in the build container (the reference is not on
the GPU box); the fixtures are committed.

    python tests/golden/make_golden.py

Fixtures
  ref_random.npz        reference random_circuit(n, depth, seed) ops + text and
                        the final state from the reference's paired-cached
                        engine (reference engine.cpp:177-238, kernel.cpp)
  ref_configs.json      for BASELINE-config circuits built by our host layer:
                        sha256 of the op bytes fed to both sides and of the
                        reference engine's final state, its norm, and samples
  test_dense_frozen.json  the reference's own frozen vector (copied verbatim
                        from reference proj/tests/test_dense.cpp:189-209)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import GATE_DTYPE, RefEngine  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402

RANDOM_CASES = [(1, 10, 2), (2, 30, 9), (3, 20, 42), (4, 30, 7), (5, 25, 1), (6, 40, 7), (7, 60, 11),
                (8, 20, 11), (8, 20, 5), (9, 80, 13), (10, 200, 3), (10, 120, 17)]

# (name, builder, args) — the circuits run through the reference engine
CONFIGS = [
    ("config0_u3_ladder_n20", "u3_ladder_circuit", (20, 20, 1)),
    ("config1_qft_n16", "qft_circuit", (16, 5)),
    ("config2_haar_sweep_n20", "haar_sweep_circuit", (20, 2508)),
    ("config3_grid_4x5_c12", "grid_circuit", (4, 5, 12, 3)),
    ("config4_u3_ladder_n18_l4", "u3_ladder_circuit", (18, 4, 4)),
]


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def build(name, fn, args):
    out = getattr(qv, fn)(*args)
    return out[0] if isinstance(out, tuple) else out


def main():
    eng = RefEngine()
    # 1. random circuits through the reference's own generator and engine
    arrays = {}
    for n, depth, seed in RANDOM_CASES:
        ops, text = eng.random_circuit(n, depth, seed)
        with eng.store(n, block_amps=4) as st:
            st.apply(ops, "paired-cached", 1, 4 * 4 * 16)
            state = st.read()
        key = f"n{n}_d{depth}_s{seed}"
        arrays[f"{key}_ops"] = np.frombuffer(ops.tobytes(), np.uint8)
        arrays[f"{key}_text"] = np.frombuffer(text.encode(), np.uint8)
        arrays[f"{key}_state"] = state
    np.savez_compressed(os.path.join(HERE, "ref_random.npz"), **arrays)

    # 2. BASELINE-config circuits (our builders) through the reference engine
    configs = {}
    for name, fn, args in CONFIGS:
        c = build(name, fn, args)
        n = c.n_qubits
        ops = np.frombuffer(c.gates().tobytes(), dtype=GATE_DTYPE)
        with eng.store(n, block_amps=1024) as st:
            st.apply(ops, "paired-cached-parallel", 4, 4 * (64 << 20))
            state = st.read()
            norm = st.norm()
        p = state.real * state.real + state.imag * state.imag
        top = sorted(range(len(p)), key=lambda i: (-p[i], i))[:8]
        configs[name] = {
            "builder": fn, "args": list(args), "n_qubits": n, "n_ops": len(c),
            "ops_sha256": sha(ops.tobytes()), "state_sha256": sha(state.tobytes()),
            "norm": norm, "first": [[a.real, a.imag] for a in state[:8]],
            "top8_index": top, "top8": [[state[i].real, state[i].imag] for i in top],
            "engine": "reference paired-cached-parallel, workers=4, block_amps=1024",
        }
    with open(os.path.join(HERE, "ref_configs.json"), "w") as f:
        json.dump(configs, f, indent=1)
    print("wrote", len(arrays) // 3, "random cases and", len(configs), "config fixtures")


if __name__ == "__main__":
    main()
