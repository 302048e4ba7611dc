"""Phase timeline of the fused tile kernel: where a tile's time goes and whether
the CTAs of one SM overlap their load, compute and store phases.

Needs the debug variant of the library (`make -C paper_2508_15545_b200 trace`
-> libqvg_trace.so, QVG_TILE_TRACE): thread 0 of the CTA that runs tile t in
[first, first + count) stamps, per launch, 24 words (TileTrace, qvg_tile.cuh):
  0 smid, 1 globaltimer at tile start, 2 clock at start, 3 clock at the end,
  4 globaltimer at the end, 5 groups, then per register group gi < 6:
  6+3gi amplitudes arrived, 7+3gi ops done, 8+3gi written back; 21 (k_tile_ahead)
  the tile's cp.async copies landed; 22 clock after the start stamps; 23 clock
  at kernel entry.

    python tools/tile_trace.py [--n 30] [--circuit config3] [--grid -1|0|1] [--count 16384] > out.json

Prints, per traced launch: [mean, p10, p90] clocks of every phase (per group:
wait = amplitudes arriving, ops, out = write-back and barrier), the CTA
preamble, and the mean number of traced CTAs resident per SM.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_15545_b200 as qv  # noqa: E402  (circuit builders only; the traced runs go through ctypes)


def circuit(name, n):
    if name == "config2":
        return qv.haar_sweep_circuit(n, 2508)
    if name == "config3":
        return qv.grid_circuit(5, 6, 24, 1) if n == 30 else qv.grid_circuit(4, n // 4, 8, 1)
    if name == "config1":
        return qv.qft_circuit(n, 1)[0]
    return qv.u3_ladder_circuit(n, 4, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--circuit", default="config3")
    ap.add_argument("--grid", type=int, default=-1)
    ap.add_argument("--count", type=int, default=16384)
    ap.add_argument("--launches", type=int, default=12)
    ap.add_argument("--opts", default="", help="key=value,... raw QVG_OPT numbers")
    a = ap.parse_args()
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2508_15545_b200", "libqvg_trace.so"))
    lib.qvg_last_error.restype = ctypes.c_char_p

    def ck(rc):
        if rc != 0:
            raise RuntimeError(lib.qvg_last_error().decode())

    st = ctypes.c_void_p()
    ck(lib.qvg_create(ctypes.c_uint32(a.n), ctypes.c_uint32(128), 0, ctypes.byref(st)))
    ck(lib.qvg_set_option(st, 14, ctypes.c_int64(0)))  # QVG_OPT_GRAPH off
    ck(lib.qvg_set_option(st, 22, ctypes.c_int64(a.grid)))  # QVG_OPT_TILE_GRID
    for kv in filter(None, a.opts.split(",")):
        k, v = kv.split("=")
        ck(lib.qvg_set_option(st, int(k), ctypes.c_int64(int(v))))
    ck(lib.qvg_init_basis(st, ctypes.c_uint64(0)))
    gates = np.frombuffer(circuit(a.circuit, a.n).gates().tobytes(), dtype=np.uint8).copy()
    count = len(circuit(a.circuit, a.n))
    gp = gates.ctypes.data_as(ctypes.c_void_p)
    ck(lib.qvg_apply(st, gp, ctypes.c_uint64(count)))  # warm-up, untraced
    ck(lib.qvg_sync(st))
    ntiles = 1 << (a.n - 11)
    first = ntiles // 2
    buf = torch.zeros(24 * a.count * a.launches, dtype=torch.int64, device="cuda")
    lib.qvg_debug_tile_trace(ctypes.c_void_p(buf.data_ptr()), ctypes.c_uint64(first), ctypes.c_uint64(a.count),
                             ctypes.c_uint64(a.launches))
    ck(lib.qvg_apply(st, gp, ctypes.c_uint64(count)))
    ck(lib.qvg_sync(st))
    torch.cuda.synchronize()
    t = buf.cpu().numpy().reshape(a.launches, a.count, 24)
    out = {"n": a.n, "circuit": a.circuit, "grid": a.grid, "count": a.count, "launches": []}
    for li in range(a.launches):
        r = t[li]
        r = r[r[:, 2] != 0]
        if len(r) == 0:
            continue
        ng = int(r[0, 5])
        f = lambda x: [round(float(np.mean(x)), 1), round(float(np.percentile(x, 10)), 1), round(float(np.percentile(x, 90)), 1)]
        groups = []
        prev = r[:, 2]
        tot = {"wait": 0.0, "ops": 0.0, "out": 0.0}
        for gi in range(min(ng, 6)):
            a_, b_, c_ = r[:, 6 + 3 * gi], r[:, 7 + 3 * gi], r[:, 8 + 3 * gi]
            groups.append({"wait": f(a_ - prev), "ops": f(b_ - a_), "out": f(c_ - b_)})
            tot["wait"] += float(np.mean(a_ - prev)); tot["ops"] += float(np.mean(b_ - a_)); tot["out"] += float(np.mean(c_ - b_))
            prev = c_
        wall_ns = float(r[:, 4].max() - r[:, 1].min())
        res = []
        for sm in np.unique(r[:, 0]):
            q = r[r[:, 0] == sm]
            if len(q) < 8:
                continue
            span = float(q[:, 3].max() - q[:, 23].min())
            res.append(float((q[:, 3] - q[:, 23]).sum()) / span)
        nsm = max(1, len(np.unique(r[:, 0])))
        out["launches"].append({
            "launch": li, "tiles": int(len(r)), "sms": int(nsm), "groups": ng,
            "us_per_tile_per_sm": wall_ns / 1e3 / (len(r) / nsm),
            "clk_tile_total": f(r[:, 3] - r[:, 23]),
            "clk_preamble": f(r[:, 2] - r[:, 23]),
            "clk_tail": f(r[:, 3] - prev),
            "clk_stamp_overhead": f(r[:, 22] - r[:, 2]),
            "clk_wait_copies": f(r[:, 21] - r[:, 22]) if np.all(r[:, 21] != 0) else None,
            "clk_sum": {k: round(v, 1) for k, v in tot.items()},
            "per_group": groups,
            "mean_resident_ctas_per_sm": float(np.mean(res)) if res else None,
        })
    print(json.dumps(out, indent=1))
    np.save(os.path.join(ROOT, "gpurun_out", f"tile_trace_{a.circuit}_g{a.grid}.npy"), t)
    lib.qvg_destroy(st)


if __name__ == "__main__":
    main()
