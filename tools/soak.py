"""Soak test of the fused planner and tile kernels against the C oracle: seeded
random circuits (the reference's generator: H/X/Z/S/T/sqrt gates, rotations,
U3, CX/CZ/CP/CU on random qubits) at n = 5..max_n, random tile shapes and
engine options, complex128 compared with np.array_equal (bit-identical values;
+-0 equal), plus structured circuits (U3 + CX ladders, grids, QFT) that drive
the planner's group reordering. Prints one JSON line; exits 1 on a mismatch.

    python tools/soak.py [--seconds 240] [--min-n 5] [--max-n 18] [--seed 1]
"""
import argparse
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402,F401

import paper_2508_15545_b200 as qv  # noqa: E402
from conftest import gate_array  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402  (the checker, tests/ and tools only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240)
    ap.add_argument("--max-n", type=int, default=18)
    ap.add_argument("--min-n", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = random.Random(a.seed)
    oracle = Oracle()
    t0 = time.time()
    cases = fails = 0
    kinds = {}
    while time.time() - t0 < a.seconds:
        n = rng.randint(a.min_n, a.max_n)
        kind = rng.choice(["random", "random", "random", "ladder", "grid", "qft", "sweep"])
        seed = rng.randrange(1 << 31)
        if kind == "random":
            c = qv.random_circuit(n, rng.randint(1, 400 if n <= 18 else 120), seed)
        elif kind == "ladder":
            c = qv.u3_ladder_circuit(n, rng.randint(1, 6), seed)
        elif kind == "grid":
            rows = rng.choice([r for r in (2, 3, 4) if n % r == 0] or [1])
            c = qv.grid_circuit(rows, n // rows, rng.randint(1, 8), seed)
        elif kind == "qft":
            c = qv.qft_circuit(n, seed)[0]
        else:
            c = qv.haar_sweep_circuit(n, seed)
        want = oracle.simulate(n, gate_array(c))
        opts = {"tile": rng.choice([0, 0, 0, 5, 7, 9, 10, 11, 12]), "sub": rng.choice([4, 4, 3]),
                "reorder": rng.choice([2, 2, 2, 0]), "pipe": rng.choice([-1, -1, 0, 5]),
                "grid": rng.choice([-1, -1, 0]), "graph": rng.choice([0, 2]), "classes": rng.choice([1, 1, 0]),
                "shards": rng.choice([1, 1, 1, 2, 4]) if n >= 8 else 1}
        st = (qv.StateVector.create(n, 128, 0) if opts["shards"] == 1
              else qv.StateVector.create_sharded(n, 128, 0, 0, opts["shards"], None))
        for key, val in ((qv.OPT_SUB_BITS, opts["sub"]), (qv.OPT_REORDER, opts["reorder"]), (qv.OPT_PIPE, opts["pipe"]),
                         (qv.OPT_TILE_GRID, opts["grid"]), (qv.OPT_GRAPH, opts["graph"]),
                         (qv.OPT_CLASSES, opts["classes"])):
            st.set_option(key, val)
        qv.apply_circuit(st, c, tile_qubits=opts["tile"])
        got = st.read_state()
        cases += 1
        kinds[kind] = kinds.get(kind, 0) + 1
        if not np.array_equal(got, want):
            fails += 1
            print(json.dumps({"mismatch": {"n": n, "kind": kind, "seed": seed, "ops": len(c), "opts": opts,
                                           "max_abs": float(np.abs(got - want).max())}}), flush=True)
            if fails >= 5:
                break
    print(json.dumps({"cases": cases, "by_kind": kinds, "mismatches": fails, "seconds": round(time.time() - t0, 1),
                      "min_n": a.min_n, "max_n": a.max_n, "seed": a.seed}))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
