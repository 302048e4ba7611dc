"""Exchange-transport A/B on one GPU with virtual shards: config 4's layer
circuit (U3 layers + CX ladder) at n qubits over G shards, with
QVG_OPT_EXCHANGE 0 (swap kernel + separate gate), 1 (k_xchg exchange only)
and 2 (k_xchg fused with the gate that triggered the exchange), pairwise
exchanges only, and batched exchanges (QVG_OPT_BATCH_EXCHANGE 4, k_mxchg).

On one device every "remote" byte is an HBM byte, so this measures the
kernels' HBM efficiency and the passes the fusion removes, not NVLink.

    python tools/xchg_ab.py [--n 30] [--layers 4] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402


def timed(st, circ, reps, fuse):
    stream = torch.cuda.ExternalStream(st.stream())
    qv.apply_circuit(st, circ, fuse=fuse)  # warm-up (and leaves the qubit map permuted, as in a long run)
    st.sync()
    st.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        qv.apply_circuit(st, circ, fuse=fuse, sync=False)
    e1.record(stream)
    st.sync()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, st.stats()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    circ = qv.u3_ladder_circuit(a.n, a.layers, 4)
    rows = []
    for world in (2, 4, 8):
        for fuse in (True, False):
            ref = None
            for mode, batch in ((0, 1), (1, 1), (2, 1), (1, 4)):
                st = qv.StateVector.create_sharded(a.n, 128, 0, 0, world, None)
                st.set_option(qv.OPT_EXCHANGE, mode)
                st.set_option(qv.OPT_BATCH_EXCHANGE, batch)
                ms, s = timed(st, circ, a.reps, fuse)
                # bit-identity across modes on the same circuit
                head = st.read_state(0, 1 << 20)
                same = None
                if ref is None:
                    ref = head
                else:
                    same = bool((head == ref).all())
                row = {"n": a.n, "world": world, "fuse": fuse, "mode": mode, "batch": batch, "ms": ms,
                       "passes": s["passes"] / a.reps, "exchanges": s["exchanges"] / a.reps,
                       "fused_exchanges": s["fused_exchanges"] / a.reps, "same_as_mode0": same}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del st
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
