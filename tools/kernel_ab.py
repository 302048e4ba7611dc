"""A/B timing of per-gate kernel variants on one device-resident state
(CUDA events on the state's stream, median of reps, interleaved variants).

    python tools/kernel_ab.py [--n 30] [--reps 10] > profiles/rNN_kernel_ab.json

Rows: every (gate, target, control) case of interest, timed with the
warp-shuffle low-target kernel on and off (QVG_OPT_LOW_KERNEL), reporting ms
and algorithmic GB/s (the planner's byte count for the pass).
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


# (name, low-target shuffle kernel, min_run bytes, predicated stores)
VARIANTS = [("pairs_run32", 0, 32, 0), ("pairs_run64", 0, 64, 0), ("pairs_run128", 0, 128, 0),
            ("pairs_run128_pred", 0, 128, 1), ("pairs_run32_pred", 0, 32, 1), ("low_run32", 1, 32, 0)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--precision", type=int, default=128)
    a = ap.parse_args()
    n = a.n
    st = qv.StateVector.create(n, a.precision, 0)
    st.set_option(qv.OPT_FUSE, 0)
    st.apply_gates(qv.make_benchmark_circuit(n).gates())
    stream = torch.cuda.ExternalStream(st.stream())
    cases = []
    for q in (0, 1, 2, 3, 4, 5, 8, 15, 29):
        cases.append((f"h {q}", f"h {q}"))
    for c, t in ((0, 1), (1, 0), (1, 2), (2, 3), (3, 4), (4, 3), (0, 15), (1, 15), (2, 15), (3, 15), (4, 15),
                 (15, 0), (15, 3), (15, 16), (29, 28), (5, 6)):
        cases.append((f"cx {c} {t}", f"cx {c} {t}"))
    for c, t in ((0, 1), (3, 20), (14, 15), (28, 29)):
        cases.append((f"cz {c} {t}", f"cz {c} {t}"))
    cases.append(("t 7", "t 7"))
    rows = []
    for name, text in cases:
        gates = qv.parse_circuit(f"qubits {n}\n{text}\n").gates()
        _, _, nbytes = qv.plan_passes(n, gates, a.precision, False)
        res = {}
        for vname, low, min_run, pred in VARIANTS:
            st.set_option(qv.OPT_LOW_KERNEL, low)
            st.set_option(qv.OPT_MIN_RUN, min_run)
            st.set_option(qv.OPT_PRED_STORE, pred)
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.apply_gates(gates, sync=False)
                e1.record(stream)
                st.sync()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            res[vname] = {"ms": ms, "gbs": nbytes / (ms / 1e3) / 1e9}
        rows.append({"op": name, "alg_bytes": nbytes, **res})
        print(f"{name:10s} " + " ".join(f"{k}={v['ms']:.2f}" for k, v in res.items()), file=sys.stderr)
    print(json.dumps({"n": n, "precision": a.precision, "reps": a.reps, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
