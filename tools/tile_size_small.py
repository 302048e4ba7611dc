"""Tile size x register subcube at small n (config 0's circuit): passes and
device ms per call.

    python tools/tile_size_small.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_15545_b200 as qv
for n in (16, 20, 22):
    c = qv.u3_ladder_circuit(n, 20, 1); g = c.gates()
    for k in (7, 8, 9, 10, 11):
        for sub in (3, 4):
            if sub == 4 and k < 7: continue
            st = qv.StateVector.create(n, 128, 0)
            st.set_option(qv.OPT_TILE_QUBITS, k); st.set_option(qv.OPT_SUB_BITS, sub)
            stream = torch.cuda.ExternalStream(st.stream())
            for _ in range(3): st.apply_gates(g)
            st.reset_stats(); ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream); st.apply_gates(g, sync=False); e1.record(stream); st.sync(); ts.append(e0.elapsed_time(e1))
            print(n, k, sub, st.stats()['passes'] / 10, round(statistics.median(ts), 3), flush=True)
# the engine's own choice (no shape option set)
for n in (12, 14, 16, 17, 18, 20):
    c = qv.u3_ladder_circuit(n, 20, 1); g = c.gates()
    st = qv.StateVector.create(n, 128, 0)
    stream = torch.cuda.ExternalStream(st.stream())
    for _ in range(3): st.apply_gates(g)
    st.reset_stats(); ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); st.apply_gates(g, sync=False); e1.record(stream); st.sync(); ts.append(e0.elapsed_time(e1))
    print(n, "auto", st.stats()['passes'] / 10, round(statistics.median(ts), 3), flush=True)
