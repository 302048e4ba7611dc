"""End-to-end pipelining A/B: host->HBM->host steps of the config-2 sweep
through the public API, with S device states on their own streams and each
PCIe copy split into C chunks (so the copy engines can interleave directions).

    python tools/e2e_ab.py [--n 30] [--steps 6]
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


def run(states, bufs, circ, steps, chunks):
    count = 1 << circ.n_qubits
    per = count // chunks
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        s, buf = states[k % len(states)], bufs[k % len(bufs)]
        for c in range(chunks):
            s.load_async(buf[c * per:(c + 1) * per], c * per)
        qv.apply_circuit(s, circ, sync=False)
        for c in range(chunks):
            s.read_async(buf[c * per:(c + 1) * per], c * per)
    for s in states:
        s.sync()
    return (time.perf_counter() - t0) * 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--states", default="2,3")
    ap.add_argument("--chunks", default="1,8")
    a = ap.parse_args()
    S_list = [int(x) for x in a.states.split(",")]
    C_list = [int(x) for x in a.chunks.split(",")]
    n = a.n
    count = 1 << n
    circ = qv.haar_sweep_circuit(n, 2508)
    bufs = []
    for _ in range(max(S_list)):
        h = torch.empty(count * 2, dtype=torch.float64, pin_memory=True)
        arr = h.numpy().view(np.complex128)
        arr[:] = 1.0 / math.sqrt(count)
        bufs.append((h, arr))
    arrs = [b[1] for b in bufs]
    states = [qv.StateVector.create(n, 128, 0) for _ in range(max(S_list))]
    out = {}
    for S in S_list:
        for C in C_list:
            run(states[:S], arrs[:S], circ, 2, C)  # warm-up
            ms = run(states[:S], arrs[:S], circ, a.steps, C)
            out[f"states{S}_chunks{C}"] = {"ms_per_step": ms, "amp_updates_per_s": len(circ) * count / (ms / 1e3)}
            print(S, C, f"{ms:.1f} ms/step", file=sys.stderr)
    print(json.dumps({"n": n, "steps": a.steps, "rows": out}, indent=1))


if __name__ == "__main__":
    main()
