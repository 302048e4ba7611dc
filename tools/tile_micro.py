"""Fused-tile micro-benchmark: one tile pass with a controlled op mix, to
separate the per-op cost from the per-group (shared-memory transpose) cost.

Each row is one circuit of `ops` dense 2x2 gates on n=28 qubits whose targets
cycle over `qubits`. It is applied as one fused pass (the planner is asked for
a single pass). The row reports ms per pass and the FP64 pipe time it implies:
28 FP64 instructions per pair at 64 lanes/clk/SM.

    python tools/tile_micro.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402
from oracle.oracle import GATE_DTYPE  # noqa: E402


def circuit(n, qubits, ops, seed=1):
    rng = np.random.default_rng(seed)
    g = np.zeros(ops, GATE_DTYPE)
    for i in range(ops):
        a = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
        q, r = np.linalg.qr(a)
        u = q * (np.diag(r) / abs(np.diag(r)))
        g[i]["kind"] = 0
        g[i]["target"] = qubits[i % len(qubits)]
        g[i]["control"] = -1
        g[i]["u"] = np.stack([u.reshape(-1).real, u.reshape(-1).imag], axis=1).reshape(-1)
    return g


def main():
    n = 28
    st = qv.StateVector.create(n, 128, 0)
    st.apply_gates(qv.make_benchmark_circuit(n).gates())
    stream = torch.cuda.ExternalStream(st.stream())
    sm_clk = 148 * 64 * 1.65e9  # FP64 lanes/s at the power-capped clock
    rows = []
    for name, qubits in [("1 group: q0-3", [0, 1, 2, 3]), ("1 group: q0,q7,q8,q9", [0, 7, 8, 9]),
                         ("3 groups: q0-10", list(range(11))), ("2 groups: q0-7", list(range(8)))]:
        for ops in (4, 16, 64):
            for sub, pf in ((3, 0), (4, 0), (4, 1)):
                g = circuit(n, qubits, ops)
                st.set_option(qv.OPT_SUB_BITS, sub)
                st.set_option(qv.OPT_PREFETCH, pf)
                st.apply_gates(g.view(np.uint8))
                st.reset_stats()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 3
                e0.record(stream)
                for _ in range(reps):
                    st.apply_gates(g.view(np.uint8), sync=False)
                e1.record(stream)
                st.sync()
                ms = e0.elapsed_time(e1) / reps
                s = st.stats()
                fp64_ms = ops * 28 * (1 << (n - 1)) / sm_clk * 1e3
                row = {"case": name, "ops": ops, "sub": sub, "prefetch": pf, "passes": s["passes"] / reps, "ms": ms,
                       "fp64_floor_ms": fp64_ms, "hbm_floor_ms": s["passes"] / reps * 2 * 16 * (1 << n) / 6.5456e12 * 1e3,
                       "fp64_frac": fp64_ms / ms}
                rows.append(row)
                print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
