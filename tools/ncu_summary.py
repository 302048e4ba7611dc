"""Summarise an ncu launch list of `bench.py` into per-kernel-class shares,
mean device time and measured DRAM traffic per launch.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -s 30 -c 120 --csv --log-file launches.csv \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e
    python tools/ncu_summary.py launches.csv --skip 30 --out profiles/rNN_bench_launches.json

Launch i (after --skip) is op (i mod 120) of the config-2 sweep, so each
launch is classified exactly like bench.py's per-kernel table.
"""
import argparse
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    launches = {}
    for r in rows:
        d = launches.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6}.get(unit, 1.0)
        d[r["Metric Name"]] = v * scale
    return [launches[k] for k in sorted(launches)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--skip", type=int, default=30, help="launches skipped by ncu -s (for op alignment)")
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--out")
    a = ap.parse_args()
    import numpy as np

    import bench
    import paper_2508_15545_b200 as qv

    recs = bench.gate_records(qv.haar_sweep_circuit(a.n, bench.SEED))
    launches = load(a.csv)
    classes = {}
    total = 0.0
    for i, L in enumerate(launches):
        op = (a.skip - 30 + i) % len(recs)
        k = bench.kernel_of(a.n, recs[op])
        t = L.get("gpu__time_duration.sum", 0.0)
        total += t
        c = classes.setdefault(k, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "alg_bytes": 0.0})
        c["launches"] += 1
        c["ms"] += t
        c["dram_bytes"] += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
        c["alg_bytes"] += bench.algorithmic_bytes(a.n, recs[op])
    out = {"source": os.path.basename(a.csv), "launches": len(launches), "total_ms": total, "classes": {}}
    for k, c in sorted(classes.items(), key=lambda kv: -kv[1]["ms"]):
        out["classes"][k] = {
            "launches": c["launches"], "share_of_step": c["ms"] / total,
            "ms_per_launch": c["ms"] / c["launches"],
            "dram_bytes_per_launch": c["dram_bytes"] / c["launches"],
            "alg_bytes_per_launch": c["alg_bytes"] / c["launches"],
            "dram_over_alg": c["dram_bytes"] / c["alg_bytes"] if c["alg_bytes"] else None,
        }
    text = json.dumps(out, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
