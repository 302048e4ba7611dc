"""A/B of the fused tile kernels: k_tile (QVG_OPT_PIPE 0, per-thread loads and
stores) against k_tile_pipe (bulk-copy producer/consumer ring, 2 or 3 stages)
on the BASELINE circuits. Device time per circuit (CUDA events on the state's
stream, median of reps), and a bitwise check that every variant leaves the
same state as k_tile (device max |delta| == 0).

    python tools/pipe_ab.py [--n 30] [--reps 3] [--precision 128] > profiles/r02_pipe_ab.json
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


def circuits(n):
    out = [("config2_haar_sweep", qv.haar_sweep_circuit(n, 2508))]
    if n == 30:
        out.append(("config3_grid_5x6_c24", qv.grid_circuit(5, 6, 24, 1)))
    out += [("config1_qft", qv.qft_circuit(n, 1)[0]), ("config0_u3_ladder_l4", qv.u3_ladder_circuit(n, 4, 1))]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", type=int, default=128)
    ap.add_argument("--pipes", default="0,2,3")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    pipes = [int(x) for x in a.pipes.split(",")]
    only = set(filter(None, a.only.split(",")))
    ref = qv.StateVector.create(a.n, a.precision, 0)
    st = qv.StateVector.create(a.n, a.precision, 0)
    stream = torch.cuda.ExternalStream(st.stream())
    rows = []
    for name, c in circuits(a.n):
        if only and name not in only:
            continue
        g = c.gates()
        row = {"circuit": name, "ops": len(c)}
        ref.set_option(qv.OPT_PIPE, 0)
        ref.init_basis(0)
        ref.apply_gates(g)
        for p in pipes:
            st.set_option(qv.OPT_PIPE, p)
            st.init_basis(0)
            st.apply_gates(g)  # warm-up, and the state compared with k_tile's
            st.sync()
            dev = st.max_deviation(ref)
            st.reset_stats()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.apply_gates(g, sync=False)
                e1.record(stream)
                st.sync()
                ts.append(e0.elapsed_time(e1))
            s = st.stats()
            ms = statistics.median(ts)
            row[f"pipe{p}"] = {"ms": ms, "passes": s["passes"] / a.reps, "max_dev_vs_k_tile": dev,
                               "hbm_gbs": s["bytes_moved"] / a.reps / (ms / 1e3) / 1e9}
        rows.append(row)
        print(name, " ".join(f"{k}={v['ms']:.2f}ms/{v['passes']:.0f}p dev={v['max_dev_vs_k_tile']:.1e}"
                             for k, v in row.items() if isinstance(v, dict)), file=sys.stderr, flush=True)
    print(json.dumps({"n": a.n, "precision": a.precision, "reps": a.reps, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
