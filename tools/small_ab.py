"""Small-state latency: config 0's circuit (U3 layers + CX ladder, 20 layers)
at small n, where a pass is a few microseconds and host-side planning and
launch cost can dominate. Reports per call: host wall time (apply + sync),
device time (CUDA events on the state's stream) and passes.

    python tools/small_ab.py [--reps 20]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("QVG_PKG_ROOT"):  # an alternative build of the package (A/B of compile-time variants)
    sys.path.insert(0, os.environ["QVG_PKG_ROOT"])

import torch  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--sizes", default="10,14,18,20,22,24")
    ap.add_argument("--graph", type=int, default=-1, help="QVG_OPT_GRAPH value to set (-1: leave default)")
    a = ap.parse_args()
    rows = []
    for n in [int(x) for x in a.sizes.split(",")]:
        c = qv.u3_ladder_circuit(n, 20, 1)
        g = c.gates()
        for fuse in (1, 0):
            st = qv.StateVector.create(n, 128, 0)
            st.set_option(qv.OPT_FUSE, fuse)
            if a.graph >= 0 and hasattr(qv, "OPT_GRAPH"):
                st.set_option(qv.OPT_GRAPH, a.graph)
            stream = torch.cuda.ExternalStream(st.stream())
            for _ in range(3):
                st.apply_gates(g)
            st.reset_stats()
            wall, dev = [], []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                e0.record(stream)
                st.apply_gates(g, sync=False)
                e1.record(stream)
                st.sync()
                wall.append((time.perf_counter() - t0) * 1e3)
                dev.append(e0.elapsed_time(e1))
            s = st.stats()
            row = {"n": n, "fuse": fuse, "ops": len(c), "passes": s["passes"] / a.reps,
                   "wall_ms": statistics.median(wall), "device_ms": statistics.median(dev)}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del st


if __name__ == "__main__":
    main()
