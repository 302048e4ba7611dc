"""FP64 rate of fused passes made of one op kind (micro-benchmark for the
tile kernels, k_tile vs the JIT kernels): n = 28, complex128, one fused pass
of `ops` identical-shape gates after a Hadamard layer. Prints device ms per
pass (CUDA events, median of reps), the FP64 instructions the pass needs per
amplitude (per op: dense 14, cmul on 1/4 of the amplitudes 1.5, ...) and the
fraction of the 64 FP64 lanes/clk/SM peak at the measured SM clock.

    python tools/diag_micro.py [--n 28] [--ops 64] [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402


def cases(n, ops):
    # (name, circuit lines, FP64 thread-instructions per amplitude for the pass)
    out = []
    out.append(("dense_u3_q0-3", [f"u3 {i % 4} 0.3 0.7 {0.1 * i}" for i in range(ops)], 14.0 * ops))
    out.append(("cp_in_group_q0-3", [f"cp {i % 4} {(i + 1) % 4} {0.1 + 0.01 * i}" for i in range(ops)], 1.5 * ops))
    out.append(("cp_ctl_outside_tile", [f"cp {12 + i % 12} {i % 4} {0.1 + 0.01 * i}" for i in range(ops)], 1.5 * ops))
    out.append(("p_target_in_group", [f"p {i % 4} {0.1 + 0.01 * i}" for i in range(ops)], 3.0 * ops))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--ops", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--jits", default="0,2")
    a = ap.parse_args()
    st = qv.StateVector.create(a.n, 128, 0)
    st.set_option(qv.OPT_GRAPH, 0)
    stream = torch.cuda.ExternalStream(st.stream())
    h = qv.parse_circuit(f"qubits {a.n}\n" + "\n".join(f"h {q}" for q in range(a.n)) + "\n").gates()
    rows = []
    for name, lines, fp64_per_amp in cases(a.n, a.ops):
        c = qv.parse_circuit(f"qubits {a.n}\n" + "\n".join(lines) + "\n").gates()
        row = {"case": name, "ops": a.ops, "fp64_per_amp": fp64_per_amp}
        for j in [int(x) for x in a.jits.split(",")]:
            st.set_option(qv.OPT_JIT, j)
            st.set_option(qv.OPT_FUSE, 0)
            st.init_basis(0)
            st.apply_gates(h)
            st.set_option(qv.OPT_FUSE, 1)
            st.apply_gates(c)
            st.sync()
            qv.jit_info(True)
            st.reset_stats()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.apply_gates(c, sync=False)
                e1.record(stream)
                st.sync()
                ts.append(e0.elapsed_time(e1))
            s = st.stats()
            ms = statistics.median(ts)
            clk = torch.cuda.clock_rate() * 1e6 if hasattr(torch.cuda, "clock_rate") else 1.9e9
            peak = 64 * 148 * clk
            row[f"jit{j}"] = {"ms": ms, "passes": s["passes"] / a.reps, "jit_passes": s["jit_passes"] / a.reps,
                              "fp64_frac": fp64_per_amp * (1 << a.n) / (ms / 1e3) / peak, "sm_clock_hz": clk}
        rows.append(row)
        print(name, {k: (round(v["ms"], 3), round(v["fp64_frac"], 3)) for k, v in row.items() if k.startswith("jit")},
              file=sys.stderr, flush=True)
    print(json.dumps({"n": a.n, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
