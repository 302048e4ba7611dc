"""Per-pass device times of the fused tile kernels WITHOUT ncu: CUPTI activity
records through torch.profiler (real concurrent execution, no replay, no clock
control), for several QVG_OPT_PIPE variants on the BASELINE circuits. For each
circuit and variant: every k_tile* launch's duration (median over reps),
the total, and per pass which variant is fastest ("best" = the sum of
per-pass minima, i.e. what a per-pass selection would give).

    python tools/pass_times.py [--n 30] [--precision 128] [--variants "jit=0;jit=2"] [--reps 3] > out.json

A variant is a ","-separated list of option=value (option = a qv.OPT_* name
without the prefix, lower case); JIT variants compile before timing.
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
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402


def circuits(n):
    out = [("config2_haar_sweep", qv.haar_sweep_circuit(n, 2508))]
    if n == 30:
        out.append(("config3_grid_5x6_c24", qv.grid_circuit(5, 6, 24, 1)))
    out += [("config1_qft", qv.qft_circuit(n, 1)[0]), ("config0_u3_ladder_l4", qv.u3_ladder_circuit(n, 4, 1))]
    return out


def kernel_times(st, g, reps):
    """[reps][passes] durations (ms) of the tile-kernel launches of one apply."""
    runs = []
    for _ in range(reps):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            st.apply_gates(g)
            st.sync()
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
              and ("k_" in e.name or "qvg_jit" in e.name)]
        ev.sort(key=lambda e: e.time_range.start)
        runs.append([(e.name, (e.time_range.end - e.time_range.start) / 1e3) for e in ev])
    return runs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--precision", type=int, default=128)
    ap.add_argument("--variants", default="jit=0;jit=2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    variants = [v.strip() for v in a.variants.split(";") if v.strip()]
    only = set(filter(None, a.only.split(",")))
    st = qv.StateVector.create(a.n, a.precision, 0)
    ref = qv.StateVector.create(a.n, a.precision, 0)  # k_tile's result (JIT off), for the bitwise check
    ref.set_option(qv.OPT_JIT, 0)
    ref.set_option(qv.OPT_GRAPH, 0)
    st.set_option(qv.OPT_GRAPH, 0)
    st.set_option(qv.OPT_TIMING, 0)
    rows = []
    for name, c in circuits(a.n):
        if only and name not in only:
            continue
        g = c.gates()
        row = {"circuit": name, "ops": len(c), "variants": {}}
        per = {}
        ref.init_basis(0)
        ref.apply_gates(g)
        for var in variants:
            st.set_option(qv.OPT_JIT, 0)
            st.set_option(qv.OPT_PIPE, 0)
            for kv in var.split(","):
                k, v = kv.split("=")
                st.set_option(getattr(qv, "OPT_" + k.strip().upper()), int(v))
            st.init_basis(0)
            st.apply_gates(g)  # warm-up (module load, JIT compiles in mode 2)
            st.sync()
            dev = st.max_deviation(ref)
            qv.jit_info(True)
            st.reset_stats()
            stream = torch.cuda.ExternalStream(st.stream())
            ev_ms = []
            for _ in range(a.reps):  # whole-circuit device time, CUDA events on the state's stream
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.apply_gates(g, sync=False)
                e1.record(stream)
                st.sync()
                ev_ms.append(e0.elapsed_time(e1))
            st.reset_stats()
            runs = kernel_times(st, g, a.reps)
            npass = min(len(r) for r in runs)  # CUPTI can drop records: use the common prefix
            names = [nm for nm, _ in runs[0][:npass]]
            ms = [statistics.median(r[i][1] for r in runs) for i in range(npass)]
            per[var] = ms
            row["variants"][var] = {"event_ms": statistics.median(ev_ms), "total_ms": sum(ms), "passes": len(ms), "pass_ms": [round(x, 4) for x in ms],
                                    "kernels": sorted(set(n.split("(")[0] for n in names)),
                                    "jit_passes": st.stats()["jit_passes"] / a.reps, "max_dev_vs_k_tile": dev}
        if len({len(v) for v in per.values()}) == 1:
            npass = len(next(iter(per.values())))
            best = [min(per[p][i] for p in variants) for i in range(npass)]
            row["best_of"] = {"total_ms": sum(best),
                              "pick": [min(variants, key=lambda p: per[p][i]) for i in range(npass)]}
        rows.append(row)
        print(name, " ".join(f"{k}={v['event_ms']:.2f}ms(cupti {v['total_ms']:.2f}/{v['passes']}) dev={v['max_dev_vs_k_tile']:.1e}"
                             for k, v in row["variants"].items()),
              f"best={row.get('best_of', {}).get('total_ms', float('nan')):.2f}", file=sys.stderr, flush=True)
    print(json.dumps({"n": a.n, "precision": a.precision, "reps": a.reps, "timing": "event_ms: CUDA events around the "
                      "circuit on the state's stream; pass_ms: CUPTI kernel activity (torch.profiler; it can miss "
                      "launches, so total_ms/passes may undercount); medians over reps", "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
