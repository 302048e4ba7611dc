"""Summarise ncu launch lists of fused circuits (tools/pass_profile.py) into
per-config HBM and FP64 figures: every pass's duration, DRAM bytes read +
written (achieved GB/s against the measured copy peak) and FP64-pipe
activity, plus the circuit totals.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\\
smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -s <n> --csv \\
        --log-file X.csv python tools/pass_profile.py --circuit grid
    python tools/fused_ncu_summary.py name=X.csv ... > profiles/rNN_fused_passes.json
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_copy_gbs", "hbm_gbs", "copy_gbs"):
            if k in d:
                return float(d[k]), "measured"
    except (OSError, ValueError):
        pass
    return 6545.6, "measured (round-1 MEASURED_PEAKS.json)"


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    d = collections.OrderedDict()
    for r in rows[1:]:
        m = d.setdefault(r[idx["ID"]], {"kernel": r[idx["Kernel Name"]]})
        unit = r[idx["Metric Unit"]]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        name = r[idx["Metric Name"]]
        if name.startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if name == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
        m[name] = v
    return list(d.values())


def main():
    pk, kind = peak()
    out = {"peak_gbs": pk, "peak_kind": kind, "configs": {}}
    for arg in sys.argv[1:]:
        name, path = arg.split("=", 1)
        passes = []
        for m in parse(path):
            ms = m["gpu__time_duration.sum"]
            b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
            passes.append({"kernel": m["kernel"].split("(")[0], "ms": round(ms, 4), "dram_gb": round(b / 1e9, 3),
                           "gbs": round(b / (ms / 1e3) / 1e9, 1), "frac_of_peak": round(b / (ms / 1e3) / 1e9 / pk, 3),
                           "fp64_pipe_pct": round(m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"], 1),
                           "issue_pct": round(m["smsp__issue_active.avg.pct_of_peak_sustained_active"], 1)})
        tot_ms = sum(p["ms"] for p in passes)
        tot_b = sum(p["dram_gb"] for p in passes) * 1e9
        out["configs"][name] = {
            "passes": len(passes), "ms": round(tot_ms, 3), "dram_gb": round(tot_b / 1e9, 2),
            "gbs": round(tot_b / (tot_ms / 1e3) / 1e9, 1), "frac_of_peak": round(tot_b / (tot_ms / 1e3) / 1e9 / pk, 3),
            "fp64_pipe_pct_time_weighted": round(sum(p["ms"] * p["fp64_pipe_pct"] for p in passes) / tot_ms, 1),
            "per_pass": passes}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
