"""The bench's e2e leg (state in from pinned host memory, fused sweep, state
out) alone, for A/B of package builds on one box: `QVG_PKG_ROOT=<dir>`
selects an alternative build (as tools/fused_ab.py).

    python tools/e2e_pkg_ab.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("QVG_PKG_ROOT"):
    sys.path.insert(0, os.environ["QVG_PKG_ROOT"])

import bench  # noqa: E402
import paper_2508_15545_b200 as qv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--reorder", type=int, default=-1)
    a = ap.parse_args()
    circ = qv.haar_sweep_circuit(30, bench.SEED)
    st = qv.StateVector.create(30, 128, 0)
    if a.reorder >= 0:
        orig = qv.StateVector.create

        def create(*args, **kw):
            s = orig(*args, **kw)
            s.set_option(qv.OPT_REORDER, a.reorder)
            return s
        qv.StateVector.create = create
        st.set_option(qv.OPT_REORDER, a.reorder)
    line = {}
    bench.e2e_leg(qv, st, circ, bench.gate_records(circ), line, argparse.Namespace(steps=a.steps))
    print(json.dumps({"pkg": os.environ.get("QVG_PKG_ROOT", "main"), "reorder": a.reorder, **line["e2e"]}))


if __name__ == "__main__":
    main()
