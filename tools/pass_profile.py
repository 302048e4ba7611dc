"""Per-pass view of a fused circuit for ncu: applies one BASELINE circuit
(fused, default options) once so that an ncu launch list shows every tile
pass with its duration, FP64-pipe and DRAM activity.

    ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\
dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active \
        -k regex:k_tile --csv python tools/pass_profile.py --circuit grid
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_15545_b200 as qv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--circuit", default="sweep", choices=["sweep", "grid", "ladder", "qft"])
    ap.add_argument("--sub", type=int, default=0, help="register subcube bits (0: the engine's default)")
    ap.add_argument("--prefetch", type=int, default=0)
    ap.add_argument("--tile", type=int, default=0, help="tile qubits (0: the precision's default)")
    ap.add_argument("--precision", type=int, default=128)
    ap.add_argument("--pipe", type=int, default=-1, help="QVG_OPT_PIPE (-1: the engine's default)")
    ap.add_argument("--jit", type=int, default=-1, help="QVG_OPT_JIT (-1: the engine's default; 2 = compile first)")
    a = ap.parse_args()
    n = a.n
    c = {"sweep": lambda: qv.haar_sweep_circuit(n, 2508),
         "grid": lambda: qv.grid_circuit(5, 6, 24, 1) if n == 30 else qv.grid_circuit(4, n // 4, 24, 1),
         "ladder": lambda: qv.u3_ladder_circuit(n, 4, 1),
         "qft": lambda: qv.qft_circuit(n, 1)[0]}[a.circuit]()
    st = qv.StateVector.create(n, a.precision, 0)
    st.set_option(qv.OPT_FUSE, 0)  # the start state: n per-gate H launches (skip them with ncu -s n)
    st.apply_gates(qv.make_benchmark_circuit(n).gates())
    st.set_option(qv.OPT_FUSE, 1)
    if a.sub:
        st.set_option(qv.OPT_SUB_BITS, a.sub)
    st.set_option(qv.OPT_PREFETCH, a.prefetch)
    if a.tile:
        st.set_option(qv.OPT_TILE_QUBITS, a.tile)
    if a.pipe >= 0:
        st.set_option(qv.OPT_PIPE, a.pipe)
    if a.jit >= 0:
        st.set_option(qv.OPT_JIT, a.jit)
    st.apply_gates(c.gates())
    st.sync()
    print("ok", st.stats())


if __name__ == "__main__":
    main()
