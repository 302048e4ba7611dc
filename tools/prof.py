"""Small profiling driver for ncu: one state, a handful of representative
gate passes (one per kernel variant), each launched separately.

  python tools/prof.py [--n 28] [--fused]
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
    ap.add_argument("--precision", type=int, default=128)
    ap.add_argument("--fused", action="store_true", help="only the fused sweep")
    ap.add_argument("--circuit", default="sweep", choices=["sweep", "grid", "ladder", "qft"])
    a = ap.parse_args()
    n = a.n
    st = qv.StateVector.create(n, a.precision, 0)
    st.apply_gates(qv.make_benchmark_circuit(n).gates())  # H on all: k_low x5 + k_pairs x(n-5)
    sweep = {"sweep": lambda: qv.haar_sweep_circuit(n, 2508),
             "grid": lambda: qv.grid_circuit(4, n // 4, 6, 1),
             "ladder": lambda: qv.u3_ladder_circuit(n, 2, 1),
             "qft": lambda: qv.qft_circuit(n, 1)[0]}[a.circuit]()
    if a.fused:
        st.set_option(qv.OPT_FUSE, 1)
        st.apply_gates(sweep.gates())
    else:
        st.set_option(qv.OPT_FUSE, 0)
        text = f"qubits {n}\nh 0\nh 12\ncx 0 1\ncx 1 0\ncx 15 0\ncx 0 15\ncx 14 15\ncz 3 20\ncp 4 9 0.3\nt 7\n"
        st.apply_gates(qv.parse_circuit(text).gates())
    st.sync()
    print("ok", st.stats())


if __name__ == "__main__":
    main()
