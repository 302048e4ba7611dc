"""Fused-pass timing on the BASELINE circuits (n=30 by default): device time
per circuit (CUDA events on the state's stream, median of reps), HBM passes,
and effective amp-updates/s, for each fused-tile variant and per-gate.

    python tools/fused_ab.py [--n 30] [--reps 3] > profiles/rNN_fused_ab.json
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("QVG_PKG_ROOT"):  # an alternative build of the package (A/B of compile-time variants)
    sys.path.insert(0, os.environ["QVG_PKG_ROOT"])

import torch  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402

# (name, fuse, sub_bits, fma, tile qubits, prefetch)
VARIANTS = [("fused_sub3_k11", 1, 3, 0, 11, 0), ("fused_sub3_k12", 1, 3, 0, 12, 0), ("fused_sub4_k12", 1, 4, 0, 12, 0),
            ("fused_sub3_k10", 1, 3, 0, 10, 0), ("fused_sub3_k11_fma", 1, 3, 1, 11, 0),
            ("fused_sub3_k11_pf", 1, 3, 0, 11, 1), ("fused_sub3_k10_pf", 1, 3, 0, 10, 1),
            ("fused_sub3_k12_pf", 1, 3, 0, 12, 1), ("fused_sub4_k11", 1, 4, 0, 11, 0),
            ("fused_reorder", 1, 4, 0, 11, 0), ("fused_sub4_k11_noclass", 1, 4, 0, 11, 0),
            ("fused_sub4_k11_inorder", 1, 4, 0, 11, 0), ("fused_sub4_k10", 1, 4, 0, 10, 0),
            ("fused_sub5_k12", 1, 5, 0, 12, 0), ("fused_sub5_k11", 1, 5, 0, 11, 0),
            ("per_gate", 0, 3, 0, 11, 0)]
# OPT_REORDER per variant: *_reorder = 1 (any commuting move, not bit-exact),
# *_inorder = 0 (circuit order), otherwise the default 2 (bit-exact moves)


def circuits(n):
    return [
        ("config2_haar_sweep", qv.haar_sweep_circuit(n, 2508)),
        ("config3_grid_5x6_c24", qv.grid_circuit(5, 6, 24, 1) if n == 30 else None),
        ("config1_qft", qv.qft_circuit(n, 1)[0]),
        ("config0_u3_ladder_l4", qv.u3_ladder_circuit(n, 4, 1)),
    ]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", type=int, default=128)
    ap.add_argument("--only", default="", help="comma-separated variant names (default: all)")
    ap.add_argument("--stage", type=int, default=-1, help="QVG_OPT_STAGE for every variant (-1: default)")
    ap.add_argument("--carriers", type=int, default=-1, help="QVG_OPT_CARRIERS for every variant (-1: default)")
    a = ap.parse_args()
    only = set(filter(None, a.only.split(",")))
    st = qv.StateVector.create(a.n, a.precision, 0)
    stream = torch.cuda.ExternalStream(st.stream())
    out = []
    for name, c in circuits(a.n):
        if c is None:
            continue
        g = c.gates()
        row = {"circuit": name, "ops": len(c)}
        for vname, fuse, sub, fma, k, pf in VARIANTS:
            if only and vname not in only:
                continue
            st.set_option(qv.OPT_TILE_QUBITS, k)
            st.set_option(qv.OPT_FUSE, fuse)
            st.set_option(qv.OPT_SUB_BITS, sub)
            st.set_option(qv.OPT_FMA, fma)
            st.set_option(qv.OPT_PREFETCH, pf)
            st.set_option(qv.OPT_REORDER, 1 if vname.endswith("reorder") else 0 if vname.endswith("inorder") else 2)
            if hasattr(qv, "OPT_CLASSES"):
                st.set_option(qv.OPT_CLASSES, 0 if vname.endswith("noclass") else 1)
            if a.stage >= 0:
                st.set_option(qv.OPT_STAGE, a.stage)
            if a.carriers >= 0:
                st.set_option(qv.OPT_CARRIERS, a.carriers)
            st.apply_gates(g)  # warm-up (and plan)
            st.reset_stats()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.apply_gates(g, sync=False)
                e1.record(stream)
                st.sync()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            s = st.stats()
            row[vname] = {"ms": ms, "passes": s["passes"] / a.reps,
                          "amp_updates_per_s": len(c) * (1 << a.n) / (ms / 1e3),
                          "hbm_gbs": s["bytes_moved"] / a.reps / (ms / 1e3) / 1e9}
        out.append(row)
        print(name, " ".join(f"{k}={v['ms']:.3f}ms/{v['passes']:.0f}p" for k, v in row.items() if isinstance(v, dict)),
              file=sys.stderr)
    st.set_option(qv.OPT_SUB_BITS, 3)
    st.set_option(qv.OPT_FMA, 0)
    st.set_option(qv.OPT_PREFETCH, 0)
    st.set_option(qv.OPT_REORDER, 2)
    st.set_option(qv.OPT_FUSE, 1)
    st.set_option(qv.OPT_TILE_QUBITS, 11)
    print(json.dumps({"n": a.n, "precision": a.precision, "reps": a.reps, "rows": out}, indent=1))


if __name__ == "__main__":
    main()
