"""Out-of-core tier against its PCIe floor: a 2^n
complex128 state in pinned host memory, config 4's U3 + CX ladder applied
through qvg_apply_host with two 2^w-amplitude HBM windows. Reports wall time,
segments (host <-> HBM streams of the whole state), host bytes moved, and
the floor: those bytes at the pinned bidirectional copy rate measured in the
same run (state-sized chunks both directions on two streams, CUDA events).

    python tools/ooc_bench.py [--n 32] [--w 30] [--layers 2] > profiles/r02_ooc.json
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402


def bidir_gbs(nbytes, chunks=8, reps=3):
    h1 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    per = nbytes // chunks
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s1)
        s2.wait_event(t0)
        for c in range(chunks):
            sl = slice(c * per, (c + 1) * per)
            with torch.cuda.stream(s1):
                d1[sl].copy_(h1[sl], non_blocking=True)
            with torch.cuda.stream(s2):
                h2[sl].copy_(d2[sl], non_blocking=True)
        e1.record(s1)
        e2.record(s2)
        torch.cuda.synchronize()
        ms = max(t0.elapsed_time(e1), t0.elapsed_time(e2))
        best = max(best, 2 * nbytes / (ms / 1e3) / 1e9)
    del h1, h2, d1, d2
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--w", type=int, default=30)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    count = 1 << a.n
    buf = torch.empty(count * 2, dtype=torch.float64, pin_memory=True)
    amps = buf.numpy().view(np.complex128)
    c = qv.u3_ladder_circuit(a.n, a.layers, 1)
    times, st = [], None
    for _ in range(a.reps):
        amps[:] = 0
        amps[0] = 1.0
        t0 = time.perf_counter()
        st = qv.apply_circuit_host(amps, c, a.w)
        times.append(time.perf_counter() - t0)
    host_bytes = st["host_bytes"]
    # the same streaming with (almost) no compute: one segment of one Z gate,
    # i.e. the sustained H2D + D2H rate of this chunk pattern
    z = qv.parse_circuit(f"qubits {a.n}\nz 0\n")
    one = []
    for _ in range(2):
        t0 = time.perf_counter()
        s1 = qv.apply_circuit_host(amps, z, a.w)
        one.append(time.perf_counter() - t0)
    seg_gbs = s1["host_bytes"] / min(one) / 1e9
    norm = float(np.sum(np.abs(amps[: 1 << 26]) ** 2))  # a slice; the full check is the tests'
    gbs = bidir_gbs(1 << 30)
    s = min(times)
    print(json.dumps({
        "n": a.n, "window_qubits": a.w, "ops": len(c), "segments": st["segments"], "passes": st["passes"],
        "host_bytes": host_bytes, "wall_s": s, "wall_all_s": times,
        "host_gbs": host_bytes / s / 1e9, "pcie_bidir_gbs": gbs,
        "pcie_floor_s": host_bytes / (gbs * 1e9), "pcie_frac": host_bytes / s / 1e9 / gbs,
        "one_segment_copy_gbs": seg_gbs, "copy_stream_frac": host_bytes / s / 1e9 / seg_gbs,
        "first_2^26_probability": norm,
        "what": "qvg_apply_host: state in pinned host memory, two HBM windows; host_bytes = H2D + D2H of every "
                "segment; floor = host_bytes at the measured pinned bidirectional rate (1 GiB chunks of a "
                "state-sized copy, both directions at once)"}, indent=1))


if __name__ == "__main__":
    main()
