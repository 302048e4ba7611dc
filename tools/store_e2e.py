"""File-level drop-in timing: apply_circuit(StateStore, circuit, strategy="gpu")
on a QVSV file (the reference's state-file format) in /dev/shm: file -> HBM,
the circuit on the device, HBM -> file. Reports the wall time split.

    python tools/store_e2e.py [--n 30]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_15545_b200 as qv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--dir", default="/dev/shm")
    a = ap.parse_args()
    path = os.path.join(a.dir, f"qvg-store-e2e-{os.getpid()}.qvs")
    try:
        t0 = time.perf_counter()
        qv.StateStore.create(path, a.n, overwrite=True)
        create_s = time.perf_counter() - t0
        c = qv.haar_sweep_circuit(a.n, 2508)
        rows = []
        for rep in range(2):
            t0 = time.perf_counter()
            m = qv.apply_circuit(qv.StateStore.open(path), c, strategy="gpu")
            wall = time.perf_counter() - t0
            rows.append({"rep": rep, "wall_s": wall, "metrics_wall_ms": m["wall_ms"],
                         "file_gb": (m["bytes_read"] + m["bytes_written"]) / 1e9,
                         "traversals": m["traversals"]})
            print(json.dumps(rows[-1]), flush=True)
        print(json.dumps({"n": a.n, "create_s": create_s, "rows": rows}))
    finally:
        if os.path.exists(path):
            os.remove(path)


if __name__ == "__main__":
    main()
