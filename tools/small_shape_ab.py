"""Tile shape at small n (graph replay on): config 0's circuit (U3 layers +
CX ladder, 20 layers), device time per apply for (tile qubits, subcube bits).
At small n a pass has too few tiles to fill 148 SMs, so the per-tile latency
(ops x subcube work per thread) sets the time, not HBM.

    python tools/small_shape_ab.py [--sizes 18,20,22,24] > profiles/r02_small_shape_ab.jsonl
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="16,18,20,22,24")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--shapes", default="11:4,11:3,10:3,10:4,9:3,12:3")
    a = ap.parse_args()
    for n in [int(x) for x in a.sizes.split(",")]:
        g = qv.u3_ladder_circuit(n, 20, 1).gates()
        for shape in a.shapes.split(","):
            k, sub = (int(x) for x in shape.split(":"))
            if k > n:
                continue
            st = qv.StateVector.create(n, 128, 0)
            st.set_option(qv.OPT_TILE_QUBITS, k)
            st.set_option(qv.OPT_SUB_BITS, sub)
            stream = torch.cuda.ExternalStream(st.stream())
            for _ in range(3):
                st.apply_gates(g)
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
            # kernel time inside one apply (CUPTI): the rest of device_ms is launch gaps
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                st.apply_gates(g)
                st.sync()
                torch.cuda.synchronize()
            ks = [(e.time_range.end - e.time_range.start) / 1e3 for e in prof.events()
                  if e.device_type == torch.autograd.DeviceType.CUDA and ("k_" in e.name or "qvg" in e.name)]
            print(json.dumps({"n": n, "tile_qubits": k, "sub": sub, "passes": s["passes"] / a.reps,
                              "graph_replays": s["graph_replays"], "device_ms": statistics.median(ts),
                              "kernel_ms_sum": sum(ks), "kernels_seen": len(ks),
                              "kernel_ms_max": max(ks) if ks else 0}), flush=True)
            del st


if __name__ == "__main__":
    main()
