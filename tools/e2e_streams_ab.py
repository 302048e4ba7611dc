"""Why the e2e step runs below the pinned bidirectional PCIe rate: the bench's
pipelined API loop (load_async / apply_circuit(sync=False) / read_async on each
state's own stream, 3 states x 8 chunks) against the same copies issued on two
dedicated copy streams (all H2D on one, all D2H on the other, ordered against
each state's stream by events), with and without the circuit, and the pure
bidirectional copy rate. n = 30 complex128 (16 GiB each way per step).

    python tools/e2e_streams_ab.py [--steps 9]
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
from cuda.bindings import runtime as rt  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402

H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
D2H = rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def api_loop(states, bufs, circ, steps, chunks):
    count = 1 << circ.n_qubits
    per = count // chunks
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        s, (_, buf) = states[k % len(states)], bufs[k % len(bufs)]
        for c in range(chunks):
            s.load_async(buf[c * per:(c + 1) * per], c * per)
        qv.apply_circuit(s, circ, sync=False)
        for c in range(chunks):
            s.read_async(buf[c * per:(c + 1) * per], c * per)
    for s in states:
        s.sync()
    return (time.perf_counter() - t0) * 1e3 / steps


def copy_streams_loop(states, bufs, circ, steps, chunks, apply=True):
    count = 1 << circ.n_qubits
    nbytes = count * 16
    per = nbytes // chunks
    sin, sout = torch.cuda.Stream(), torch.cuda.Stream()
    sts = [torch.cuda.ExternalStream(s.stream()) for s in states]
    ptrs = [s.device_buffer()[0] for s in states]
    done_out = [None] * len(states)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        i = k % len(states)
        s, st, dptr, (h, _) = states[i], sts[i], ptrs[i], bufs[i]
        hptr = h.data_ptr()
        if done_out[i] is not None:
            sin.wait_event(done_out[i])  # the state's previous result has left
        for c in range(chunks):
            rt.cudaMemcpyAsync(dptr + c * per, hptr + c * per, per, H2D, sin.cuda_stream)
        loaded = torch.cuda.Event()
        loaded.record(sin)
        st.wait_event(loaded)
        if apply:
            qv.apply_circuit(s, circ, sync=False)
        applied = torch.cuda.Event()
        applied.record(st)
        sout.wait_event(applied)
        for c in range(chunks):
            rt.cudaMemcpyAsync(hptr + c * per, dptr + c * per, per, D2H, sout.cuda_stream)
        done_out[i] = torch.cuda.Event()
        done_out[i].record(sout)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--steps", type=int, default=9)
    ap.add_argument("--chunks", type=int, default=8)
    a = ap.parse_args()
    count = 1 << a.n
    circ = qv.haar_sweep_circuit(a.n, 2508)
    bufs = []
    for _ in range(3):
        h = torch.empty(count * 2, dtype=torch.float64, pin_memory=True)
        arr = h.numpy().view(np.complex128)
        arr[:] = 1.0 / math.sqrt(count)
        bufs.append((h, arr))
    states = [qv.StateVector.create(a.n, 128, 0) for _ in range(3)]
    for s in states:  # warm the plan / graph caches
        qv.apply_circuit(s, circ)
        qv.apply_circuit(s, circ)
    out = {"n": a.n, "steps": a.steps, "chunks": a.chunks, "bytes_per_step": 2 * count * 16}
    out["api_3states_ms"] = api_loop(states, bufs, circ, a.steps, a.chunks)
    out["copy_streams_ms"] = copy_streams_loop(states, bufs, circ, a.steps, a.chunks)
    out["copy_streams_no_apply_ms"] = copy_streams_loop(states, bufs, circ, a.steps, a.chunks, apply=False)
    out["api_3states_again_ms"] = api_loop(states, bufs, circ, a.steps, a.chunks)
    for k in [x for x in out if x.endswith("_ms")]:
        out[k.replace("_ms", "_gbs")] = out["bytes_per_step"] / (out[k] / 1e3) / 1e9
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
