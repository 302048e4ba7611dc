"""Exchange kernels for ncu on one GPU (virtual shards: every "remote" byte is
an HBM byte here): k_xchg (pairwise, exchange only and fused with its gate)
and k_mxchg (batched, 2 global qubits at 4 shards).

    python tools/prof_xchg.py [--n 28]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_15545_b200 as qv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    a = ap.parse_args()
    n = a.n
    u = qv.make_gate("h")
    for world, mode, batch, text in [
        (2, 1, 1, f"h {n - 1}\n"),                      # k_xchg, exchange only
        (2, 2, 1, f"h {n - 1}\n"),                      # k_xchg fused with the H
        (4, 1, 4, f"h {n - 1}\nh {n - 2}\n"),           # k_mxchg, k = 2
    ]:
        st = qv.StateVector.create_sharded(n, 128, 0, 0, world, None)
        st.set_option(qv.OPT_EXCHANGE, mode)
        st.set_option(qv.OPT_BATCH_EXCHANGE, batch)
        st.set_option(qv.OPT_FUSE, 0)
        qv.apply_circuit(st, qv.parse_circuit(f"qubits {n}\n{text}"))
        st.sync()
        print(world, mode, batch, st.stats())
        del st


if __name__ == "__main__":
    main()
