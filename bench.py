#!/usr/bin/env python
"""Benchmark of the gate-application hot path (BASELINE.json metric:
amplitude-updates/s and HBM GB/s (% roofline) per gate pass, n=30 complex128).

Workload (BASELINE config 2): the n=30 gate-throughput sweep —
one Haar-random U on every qubit q = 0..29, then CX on every ordered pair with
|c - t| in {1, 15, 29} (120 gate passes). One "step" = one full sweep over the
device-resident 16 GiB state, one HBM pass per gate (fusion off: the metric is
per gate pass). amp-updates per pass = 2^n (the reference's one traversal per
gate, reference kernel.hpp:58-62), so value = 120 * 2^30 / t_step.
With N > 1 (torchrun), the state is sharded with 2^30 amplitudes per GPU
(n = 30 + log2 N, weak scaling) and the sweep runs at width n; gates on the
top log2 N qubits trigger NVLink half-shard exchanges.

  --impl ours (default)  libqvg.so kernels
  --impl reference       the reference's own CPU engine (oracle/_ref, compiled
                         from /root/reference by oracle/Makefile) on the host
                         cores, on a bounded sample of the same sweep: one
                         sweep gate per step in a fixed stratified order
                         (U q, then 3 CX) that keeps the sweep's 1:3 mix
                         exactly every 4 steps. It never imports the package:
                         the 120 gate records come from the committed
                         tests/golden/config2_haar_sweep_n30_ops.npy (sha256
                         pinned in tests/golden/ref_full.json and checked
                         against the package's builder by a CPU test).

  --gpus N               N > 1 needs torchrun (one rank per GPU); without
                         WORLD_SIZE the script re-launches itself under
                         torch.distributed.run when N GPUs are visible, and
                         fails (exit 2) when they are not.

Inputs are synthetic and seeded (no dataset exists for this path); the state
(16 GiB) is larger than L2 (126 MB), so no flush is needed between passes.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_QUBITS = 30
SEED = 2508
WORKLOAD = "config2: n=30 c128 sweep, Haar U on q=0..29 + CX for |c-t| in {1,15,29} (120 gate passes)"
METRIC = "amplitude-updates/s per gate pass (n=30 c128 gate sweep)"
UNIT = "amp-updates/s"
E2E_STATES = 3
E2E_CHUNKS = 8


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region
    (the profiling recipe's clocks line)."""

    NAMES = {
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, device=0, period=0.1):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period, self.stop_evt = period, threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self.stop_evt.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_traffic(kernel_class):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel
    class, from the newest ncu launch-list summary committed under profiles/
    (tools/ncu_summary.py). None when no capture exists."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_bench_launches.json")))
    for path in reversed(files):
        try:
            with open(path) as f:
                c = json.load(f)["classes"].get(kernel_class)
            if c:
                return c["dram_bytes_per_launch"], os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def gate_records(circuit):
    raw = np.frombuffer(circuit.gates().tobytes(), dtype=np.uint8)
    return raw.reshape(len(circuit), 80)


def algorithmic_bytes(n, rec, S=16):
    """Bytes one pass must move: dense 1q 2*2^n*S; controlled
    non-diagonal 2*2^(n-1)*S (sector-rounded when the control is bit 0)."""
    kind = int(np.frombuffer(rec[:4].tobytes(), np.uint32)[0])
    if kind == 0:
        return 2 * (1 << n) * S
    control = int(np.frombuffer(rec[8:12].tobytes(), np.int32)[0])
    run = (1 << control) * S
    b = 2 * (1 << (n - 1)) * S
    return min(b * max(1, 32 // run) if run < 32 else b, 2 * (1 << n) * S)


def granule_bytes(n, rec, S=16):
    """DRAM bytes a pass costs at the HBM3e access granularity measured with
    ncu (profiles/r01_ncu_summary.md, per-gate rows): reads move whole 128-B
    granules, writes 32-B sectors. A CX whose control-1 runs are 32 or 64 B
    (control qubit 1 or 2 in complex128) therefore reads the whole state while
    writing half; SURVEY §8d's sector rounding charges only half the reads."""
    total = (1 << n) * S
    kind = int(np.frombuffer(rec[:4].tobytes(), np.uint32)[0])
    if kind == 0:
        return 2 * total
    run = (1 << int(np.frombuffer(rec[8:12].tobytes(), np.int32)[0])) * S
    read = total if run < 128 else total // 2
    write = total if run < 32 else total // 2
    return read + write


def gate_label(rec):
    """'U q' for a single-qubit op, 'CX c->t' style for a controlled one."""
    kind, target = (int(x) for x in np.frombuffer(rec[:8].tobytes(), np.uint32))
    control = int(np.frombuffer(rec[8:12].tobytes(), np.int32)[0])
    return f"U {target}" if kind == 0 else f"C{control}->{target}"


def kernel_of(n, rec):
    """Launch class of a per-gate pass: every sweep op runs k_pairs (the
    warp-shuffle k_low is off by default, profiles/r01_kernel_ab.json);
    controlled ops enumerate only control=1 pairs."""
    kind = int(np.frombuffer(rec[:4].tobytes(), np.uint32)[0])
    return "k_pairs<double,4>" + ("/ctrl" if kind == 1 else "/dense")


def run_ours(args, rank, world, dist):
    import torch

    import paper_2508_15545_b200 as qv

    g = int(math.log2(world))
    n = N_QUBITS + g
    torch.cuda.set_device(0 if world == 1 else int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.cuda.current_device()
    circ = qv.haar_sweep_circuit(n, SEED)
    recs = gate_records(circ)
    nops = len(recs)
    if world == 1:
        st = qv.StateVector.create(n, 128, dev)
    elif dist is None:  # virtual shards on one device: the N > 1 code path without NCCL (tools/bench_virtual.py)
        st = qv.StateVector.create_sharded(n, 128, dev, 0, world, None)
    else:
        nid = qv.nccl_unique_id() if rank == 0 else None
        box = [nid]
        dist.broadcast_object_list(box, src=0)
        st = qv.StateVector.create_sharded(n, 128, dev, rank, world, box[0])
    st.set_option(qv.OPT_FUSE, 0)
    if world > 1:  # CUDA events around every local-pass batch and every exchange (per rank)
        st.set_option(qv.OPT_TIMING, 1)
    stream = torch.cuda.ExternalStream(st.stream(), device=dev)
    L = n - g
    # uniform start state with |a|^2 = 2^-n so no pass sees denormals/zeros
    st.apply_gates(qv.make_benchmark_circuit(n).gates())

    # N = 1: one call per gate pass, with an event after each (per-gate times).
    # N > 1: the whole sweep per call, so the shard schedule sees every op and
    # batches its global-qubit exchanges (one op per call would swap a global
    # qubit in without lookahead, then often swap it back).
    all_gates = circ.gates()

    def one_step(events=None):
        if world > 1:
            st.apply_gates(all_gates, sync=False)
            return
        for i in range(nops):
            st.apply_gates(recs[i], sync=False)
            if events is not None:
                events[i + 1].record(stream)

    for _ in range(args.warmup):
        one_step()
    st.sync()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    st.reset_stats()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nops + 1)] for _ in range(args.steps)]
    sampler = ClockSampler(dev)
    with sampler:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            evs[k][0].record(stream)
            one_step(evs[k])
        t_end.record(stream)
        st.sync()
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    stats = st.stats()
    # N = 1: per-launch durations from the interleaved events (same stream).
    # N > 1: one call per step, timed per segment by the engine (local pass
    # batches -> kernel_ms, exchanges -> exchange_ms); no per-gate times.
    per_op = np.zeros((args.steps, nops))
    if world == 1:
        for k in range(args.steps):
            for i in range(nops):
                per_op[k, i] = evs[k][i].elapsed_time(evs[k][i + 1])
    if dist is not None:
        t = torch.tensor([total_ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    value = nops * (1 << n) / (ms_step / 1e3)
    hbm_peak, peak_kind = peaks()
    local_bytes = [algorithmic_bytes(L, recs[i]) for i in range(nops)]
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128 (f64)",
        "data": "synthetic (seeded Haar-random unitaries, mt19937_64 seed 2508)",
        "config": bench_config(n, L, world),
        "gpu_launches": int(stats["kernel_launches"]),
        "clocks": sampler.summary(),
    }
    if world == 1:
        kernels = [kernel_of(L, recs[i]) for i in range(nops)]
        mean_op = per_op.mean(axis=0)
        share = {}
        for i in range(nops):
            share.setdefault(kernels[i], [0.0, 0, 0])
            share[kernels[i]][0] += mean_op[i]
            share[kernels[i]][1] += local_bytes[i]
            share[kernels[i]][2] += 1
        dom = max(share, key=lambda k: share[k][0])
        dom_ms, dom_bytes, dom_n = share[dom]
        achieved = (dom_bytes / dom_n) / ((dom_ms / dom_n) / 1e3) / 1e9
        traffic, traffic_src = measured_traffic(dom)
        for i in range(nops):  # per-op diagnostics (stderr): ms and algorithmic GB/s
            print(f"op {i:3d} {kernels[i]:24s} {mean_op[i]:8.3f} ms {local_bytes[i] / (mean_op[i] / 1e3) / 1e9:8.1f} GB/s",
                  file=sys.stderr)
        gran = [granule_bytes(L, recs[i]) for i in range(nops)]
        dense = [i for i in range(nops) if kernels[i].endswith("/dense")]
        t_dense = float(np.mean([mean_op[i] for i in dense]))
        line.update({
            "hbm_gbs_step": sum(local_bytes) / (mean_op.sum() / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm_peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": dom_bytes / dom_n,
                         "launch_ms": dom_ms / dom_n, "share_of_step": dom_ms / mean_op.sum()},
            # "quote the headline on dense 1q gates, where every
            # definition coincides" (2^n amp-updates and 2*2^n*S bytes per pass)
            "dense_1q": {"value": (1 << n) / (t_dense / 1e3), "unit": UNIT, "passes": len(dense),
                         "ms_per_pass": t_dense, "gbs": 2 * (1 << n) * 16 / (t_dense / 1e3) / 1e9,
                         "frac": 2 * (1 << n) * 16 / (t_dense / 1e3) / 1e9 / hbm_peak},
            "per_kernel": {k: {"launches_per_step": v[2], "ms_per_launch": v[0] / v[2],
                               "gbs": (v[1] / v[2]) / ((v[0] / v[2]) / 1e3) / 1e9} for k, v in share.items()},
            # per-gate time and HBM GB/s, individually;
            # granule-rounded bytes beside the sector-rounded ones where they differ
            "per_gate": [dict({"op": i, "gate": gate_label(recs[i]), "ms": round(float(mean_op[i]), 4),
                               "gbs": round(local_bytes[i] / (mean_op[i] / 1e3) / 1e9, 1)},
                              **({"granule_gbs": round(gran[i] / (mean_op[i] / 1e3) / 1e9, 1),
                                  "granule_frac": round(gran[i] / (mean_op[i] / 1e3) / 1e9 / hbm_peak, 3)}
                                 if gran[i] != local_bytes[i] else {})) for i in range(nops)],
            "per_gate_timing": "CUDA events between launches on the state's stream",
            "granule_note": "granule_gbs: DRAM bytes at the measured access granularity (128-B reads, 32-B "
                            "writes): CX with control qubit 1/2 (32/64-B runs) read the whole state",
        })
    else:
        t = torch.tensor([stats["kernel_ms"] / args.steps, stats["exchange_ms"] / args.steps,
                          stats["exchange_bytes"] / args.steps, stats["bytes_moved"] / args.steps],
                         dtype=torch.float64, device=f"cuda:{dev}")
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        k_ms, x_ms, x_bytes, hbm_bytes = (float(v) for v in t.tolist())
        local_gbs = hbm_bytes / (k_ms / 1e3) / 1e9 if k_ms else None
        x_gbs = x_bytes / (x_ms / 1e3) / 1e9 if x_ms else None
        line.update({
            # measured per rank with CUDA events around every local-pass batch
            # (max over ranks); no per-gate split at N > 1
            "roofline": {"bound": "hbm", "kernel": "local gate passes (all k_pairs classes, per rank)",
                         "achieved": local_gbs, "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": local_gbs / hbm_peak if local_gbs else None, "traffic": None,
                         "local_ms_per_step": k_ms, "share_of_step": k_ms / ms_step if ms_step else None},
            "per_gate": None,
            "per_gate_timing": "N > 1: the whole sweep per call (exchange lookahead); segments timed by the "
                               "engine (QVG_OPT_TIMING), not per gate",
            "exchanges_per_step": stats["exchanges"] / args.steps,
            "exchange": {"bound": "nvlink", "bytes_per_step_per_gpu": x_bytes, "ms_per_step": x_ms,
                         "gbs_per_gpu": x_gbs, "peak_gbs": 900.0,
                         "peak_kind": "NVLink 5 per direction per GPU (north_star)",
                         "frac": x_gbs / 900.0 if x_gbs else None,
                         "frac_of_measured_peer_copy": x_gbs / 770.0 if x_gbs else None,
                         "transport": "peer-memory kernel (CUDA IPC) when peers map, else NCCL copy"},
        })
    return st, circ, recs, line, n


def bench_config(n, L, world):
    """The `config` object both arms print (same keys, same values)."""
    return {"workload": WORKLOAD if world == 1 else WORKLOAD.replace("n=30", f"n={n}"),
            "n_qubits": n, "local_qubits": L, "precision": "complex128", "gate_passes_per_step": 120,
            "fusion": "off (one HBM pass per gate)", "l2": "state 16 GiB/GPU >> 126 MB L2; no flush needed",
            "parallelism": f"shard{world}"}


def fused_leg(qv, st, circ, line, args):
    """The same sweep through the fused planner (not the headline: the metric
    is per gate pass)."""
    import torch

    st.set_option(qv.OPT_FUSE, 1)
    stream = torch.cuda.ExternalStream(st.stream())
    for _ in range(2):  # the second apply of a repeated circuit captures its CUDA graph (QVG_OPT_GRAPH auto)
        st.apply_gates(circ.gates())
    st.sync()
    st.reset_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    reps = max(1, args.steps)
    for _ in range(reps):
        st.apply_gates(circ.gates(), sync=False)
    b.record(stream)
    st.sync()
    ms = a.elapsed_time(b) / reps
    s = st.stats()
    hbm = s["bytes_moved"] / reps / (ms / 1e3) / 1e9
    line["fused"] = {"ms_per_step": ms, "value": len(circ) * (1 << circ.n_qubits) / (ms / 1e3),
                     "passes_per_step": s["passes"] / reps, "fused_passes_per_step": s["fused_passes"] / reps,
                     "hbm_gbs": hbm, "hbm_frac": hbm / peaks()[0],
                     "note": "tile passes (k_tile / k_tile_ahead): per-pass DRAM, FP64 and issue figures in profiles/r02_fused_passes.json"}
    st.set_option(qv.OPT_FUSE, 0)


def c64_leg(qv, circ, recs, line, args):
    """BASELINE config 2 also names complex64: the same per-gate sweep on an
    8 GiB complex64 state (fusion off, per-launch events on the state's
    stream), its dominant launch class against the HBM roofline, per-gate ms
    and GB/s, and the fused time. Not the headline (the metric is c128)."""
    import torch

    n = circ.n_qubits
    nops = len(recs)
    st = qv.StateVector.create(n, 64, torch.cuda.current_device())
    st.set_option(qv.OPT_FUSE, 0)
    stream = torch.cuda.ExternalStream(st.stream())
    st.apply_gates(qv.make_benchmark_circuit(n).gates())
    for _ in range(args.warmup):
        for i in range(nops):
            st.apply_gates(recs[i], sync=False)
    st.sync()
    steps = max(1, args.steps)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nops + 1)] for _ in range(steps)]
    for k in range(steps):
        evs[k][0].record(stream)
        for i in range(nops):
            st.apply_gates(recs[i], sync=False)
            evs[k][i + 1].record(stream)
    st.sync()
    per_op = np.array([[evs[k][i].elapsed_time(evs[k][i + 1]) for i in range(nops)] for k in range(steps)])
    mean_op = per_op.mean(axis=0)
    ms_step = float(per_op.sum(axis=1).mean())
    nbytes = [algorithmic_bytes(n, recs[i], S=8) for i in range(nops)]
    share = {}
    for i in range(nops):
        k = kernel_of(n, recs[i]).replace("double", "float")
        share.setdefault(k, [0.0, 0, 0])
        share[k][0] += mean_op[i]
        share[k][1] += nbytes[i]
        share[k][2] += 1
    dom = max(share, key=lambda k: share[k][0])
    dom_ms, dom_bytes, dom_n = share[dom]
    hbm_peak, peak_kind = peaks()
    achieved = (dom_bytes / dom_n) / ((dom_ms / dom_n) / 1e3) / 1e9
    st.set_option(qv.OPT_FUSE, 1)
    for _ in range(2):  # eager, then graph capture (QVG_OPT_GRAPH auto)
        st.apply_gates(circ.gates())
    st.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        st.apply_gates(circ.gates(), sync=False)
    b.record(stream)
    st.sync()
    fused_ms = a.elapsed_time(b) / steps
    line["c64"] = {
        "value": nops * (1 << n) / (ms_step / 1e3), "unit": UNIT, "ms_per_step": ms_step, "dtype": "c64 (f32)",
        "hbm_gbs_step": sum(nbytes) / (ms_step / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": achieved / hbm_peak, "launch_ms": dom_ms / dom_n,
                     "algorithmic_bytes_per_launch": dom_bytes / dom_n},
        "per_kernel": {k: {"launches_per_step": v[2], "ms_per_launch": v[0] / v[2],
                           "gbs": (v[1] / v[2]) / ((v[0] / v[2]) / 1e3) / 1e9} for k, v in share.items()},
        "per_gate": [{"op": i, "gate": gate_label(recs[i]), "ms": round(float(mean_op[i]), 4),
                      "gbs": round(nbytes[i] / (mean_op[i] / 1e3) / 1e9, 1)} for i in range(nops)],
        "fused": {"ms_per_step": fused_ms, "value": nops * (1 << n) / (fused_ms / 1e3)},
    }
    del st


def pcie_bidir_gbs(host, host2, chunks=E2E_CHUNKS):
    """The e2e roofline: pinned host<->device bandwidth with both directions
    busy at once, measured the way the e2e step moves data — the state-sized
    buffer in `chunks` cudaMemcpyAsync pieces per direction on two streams,
    timed with CUDA events (start on one stream, the other waits on it; end =
    the later of the two streams' end events). Best of 3."""
    import torch

    nbytes = host.numel() * host.element_size()
    h = host.view(torch.uint8)
    h2 = host2.view(torch.uint8)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    per = nbytes // chunks
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s1)
        s2.wait_event(t0)
        for c in range(chunks):
            sl = slice(c * per, (c + 1) * per if c + 1 < chunks else nbytes)
            with torch.cuda.stream(s1):
                d[sl].copy_(h[sl], non_blocking=True)
            with torch.cuda.stream(s2):
                h2[sl].copy_(d2[sl], non_blocking=True)
        e1.record(s1)
        e2.record(s2)
        torch.cuda.synchronize()
        ms = max(t0.elapsed_time(e1), t0.elapsed_time(e2))
        best = max(best, 2 * nbytes / (ms / 1e3) / 1e9)
    del d, d2
    return best


def e2e_leg(qv, st, circ, recs, line, args):
    """The same metric through the public API with HOST buffers: every step
    copies a 16 GiB state from pinned host memory to the device, runs the sweep
    with the API's defaults (`apply_circuit(state, circuit)`: strategy gpu,
    fusion on) and copies the state back, all inside the timed region.

    value: a stream of independent steps over E2E_STATES device states on their
    own streams (load_async / apply_circuit(sync=False) / read_async), so one
    state's PCIe copies overlap another's gates (PCIe is full duplex).
    latency_ms: one step alone, synchronous (load_state / apply_circuit /
    read_into)."""
    import torch

    n = circ.n_qubits
    count = 1 << n
    bufs = []
    for _ in range(E2E_STATES):
        h = torch.empty(count * 2, dtype=torch.float64, pin_memory=True)
        a = h.numpy().view(np.complex128)
        a[:] = 1.0 / math.sqrt(count)
        bufs.append((h, a))
    # serial latency of one step (best of 2)
    latency = float("inf")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.load_state(bufs[0][1])
        m = qv.apply_circuit(st, circ)
        st.read_into(bufs[0][1])
        latency = min(latency, (time.perf_counter() - t0) * 1e3)
    # pipelined stream of steps over E2E_STATES device states, each copy in
    # E2E_CHUNKS pieces so the copy engines interleave H2D and D2H
    # (profiles/r01_e2e_ab.json: 3 states x 8 chunks 416 ms/step, 2 x 1 472)
    states = [st] + [qv.StateVector.create(n, 128, 0) for _ in range(E2E_STATES - 1)]
    steps = max(2 * E2E_STATES, args.steps)
    per = count // E2E_CHUNKS

    def stream_of_steps(apply):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(steps):
            s, (_, buf) = states[k % E2E_STATES], bufs[k % E2E_STATES]
            for c in range(E2E_CHUNKS):
                s.load_async(buf[c * per:(c + 1) * per], c * per)
            if apply:
                qv.apply_circuit(s, circ, sync=False)
            for c in range(E2E_CHUNKS):
                s.read_async(buf[c * per:(c + 1) * per], c * per)
        for s in states:
            s.sync()
        return (time.perf_counter() - t0) * 1e3 / steps

    ms = stream_of_steps(True)
    # the same stream of copies with no circuit: the sustained floor of this
    # H2D + D2H pattern (tools/e2e_streams_ab.py: dedicated copy streams are
    # no faster, profiles/r02_e2e_streams.json)
    copy_ms = stream_of_steps(False)
    del states[1:]
    pcie = pcie_bidir_gbs(bufs[0][0], bufs[1][0])
    line["e2e"] = {"value": len(circ) * count / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
                   "pcie_bidir_gbs": pcie, "pcie_frac": (2 * count * 16 / (ms / 1e3) / 1e9) / pcie,
                   "copy_only_ms_per_step": copy_ms, "copy_only_frac": copy_ms / ms,
                   # one request alone, synchronous: load -> apply -> read
                   "serial": {"value": len(circ) * count / (latency / 1e3), "unit": UNIT, "ms": latency},
                   "steps": steps, "h2d_bytes_per_step": count * 16, "d2h_bytes_per_step": count * 16,
                   "hbm_passes_per_step": m["traversals"],
                   "path": "per step: StateVector.load_async(pinned) -> apply_circuit(state, circuit) [API defaults: "
                           f"gpu, fused] -> read_async(pinned); {E2E_STATES} states rotate (pipelined throughput), "
                           f"copies in {E2E_CHUNKS} chunks, host wall clock; `serial` = one step alone"}


def e2e_leg_sharded(qv, st, circ, line, args, rank, world, dist):
    """e2e at N > 1: every rank copies its own 2^L-amplitude shard from pinned
    host memory, the sweep runs through `apply_circuit(state, circuit)` (API
    defaults: fused, exchanges over NCCL/NVLink), and every rank reads its
    shard back (the read restores the canonical qubit order first). One state
    per rank, steps back to back; the step time is the max over ranks."""
    import torch

    n = circ.n_qubits
    L = n - int(math.log2(world))
    local = 1 << L
    h = torch.empty(local * 2, dtype=torch.float64, pin_memory=True)
    buf = h.numpy().view(np.complex128)
    buf[:] = 1.0 / math.sqrt(1 << n)
    off = rank * local
    steps = max(2, args.steps)
    st.set_option(qv.OPT_FUSE, 1)
    m = None
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        st.load_async(buf, off)
        m = qv.apply_circuit(st, circ, sync=False)
        st.read_async(buf, off)
        st.sync()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    t = torch.tensor([ms], device=f"cuda:{torch.cuda.current_device()}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    st.set_option(qv.OPT_FUSE, 0)
    line["e2e"] = {"value": len(circ) * (1 << n) / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
                   "h2d_bytes_per_step": (1 << n) * 16, "d2h_bytes_per_step": (1 << n) * 16,
                   "hbm_passes_per_step": m["traversals"] if m else None,
                   "path": f"per step on each of {world} ranks: load_async(own pinned shard) -> apply_circuit(state, "
                           "circuit) [API defaults: gpu, fused, exchanges] -> read_async(own shard); "
                           "wall clock, max over ranks; bytes are whole-job totals"}


SWEEP_OPS = os.path.join(ROOT, "tests", "golden", "config2_haar_sweep_n30_ops.npy")
SWEEP_FIXTURE = os.path.join(ROOT, "tests", "golden", "ref_full.json")


def sweep_ops():
    """The config-2 sweep's 120 qvg_gate records (Haar U on q = 0..29, then 90
    CX) from the committed fixture — the reference arm and the cpu_baseline
    leg never import the package. sha256 pinned in ref_full.json (and
    tests/test_oracle.py checks the package's builder emits the same bytes)."""
    import hashlib

    from oracle.oracle import GATE_DTYPE

    ops = np.load(SWEEP_OPS)
    with open(SWEEP_FIXTURE) as f:
        want = json.load(f)["config2_haar_sweep_n30"]["ops_sha256"]
    if hashlib.sha256(ops.tobytes()).hexdigest() != want:
        raise RuntimeError(f"{SWEEP_OPS} does not match its pinned sha256")
    return np.ascontiguousarray(ops, GATE_DTYPE)


def stratified_order(n_u=30, n_cx=90):
    """Gate order for one-gate steps that keeps the sweep's 1 U : 3 CX mix
    exactly in every 4 consecutive steps: U0, CX0, CX1, CX2, U1, CX3, ...
    (indices into the sweep; a full cycle is the whole sweep once)."""
    per = n_cx // n_u
    order = []
    for q in range(n_u):
        order.append(q)
        order += [n_u + per * q + j for j in range(per)]
    return order


def ref_store_ok(scratch, n):
    try:
        st_ = os.statvfs(scratch)
        return st_.f_bavail * st_.f_frsize >= (16 << n) * 1.1
    except OSError:
        return True


def cpu_baseline(args):
    """The reference engine (oracle/_ref) on the host cores: a bounded sample of
    the same n=30 sweep — its first 4 gates in the stratified order (Haar U on
    q=0 and the CX 0->1, 0->15, 0->29: the sweep's 1:3 mix), strategy
    paired-cached-parallel, workers = host cores, block 65536, cache
    workers x 64 MiB, store on /dev/shm (the reference's RAM-disk setup)."""
    from oracle.oracle import RefEngine, default_scratch

    if not RefEngine.available():
        return None
    eng = RefEngine()
    n = N_QUBITS
    cores = os.cpu_count() or 1
    scratch = default_scratch()
    if not ref_store_ok(scratch, n):
        return {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"skipped: {scratch} has < 17.6 GB free for the n=30 store"}
    ops = sweep_ops()
    sample = ops[stratified_order()[:4]]
    with eng.store(n, 65536, 0, scratch) as store:
        store.apply(sample[:1], "paired-cached-parallel", cores, cores * (64 << 20))  # touch every page
        wall = store.apply(sample, "paired-cached-parallel", cores, cores * (64 << 20))
        # also the single-threaded column (the paper's 1-worker
        # paired_cached with a 64 MiB window), one gate pass
        single = store.apply(sample[:1], "paired-cached", 1, 64 << 20)
    return {"value": len(sample) * (1 << n) / (wall / 1e3), "unit": UNIT, "cores": cores, "kind": "reference",
            "ms_per_gate": wall / len(sample),
            "sample": "4 gate passes of the n=30 sweep (Haar U q=0, CX 0->1, 0->15, 0->29: the sweep's 1:3 mix), "
                      f"paired-cached-parallel, workers={cores}, block_amps=65536, store on {scratch}",
            "single_thread": {"value": (1 << n) / (single / 1e3), "unit": UNIT, "cores": 1, "ms_per_gate": single,
                              "sample": "1 gate pass (Haar U q=0), paired-cached, 1 worker, 64 MiB window"}}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU engine (oracle/_ref) on the
    host cores, through its public apply_circuit with a QVSV store on
    /dev/shm. One sweep gate per step in stratified_order (the sweep's exact
    1:3 U:CX mix every 4 steps; the timed steps start at the cycle's start),
    value = amp-updates per gate pass / time, the same metric, unit and config
    object as our arm. Rank 0 only under torchrun; the state is n = 30 for
    every N (the CPU holds one 16 GiB store)."""
    from oracle.oracle import RefEngine, default_scratch

    if rank != 0:
        return None
    if not RefEngine.available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libqvsim_ref.so not built (needs /root/reference)"}
    eng = RefEngine()
    n = N_QUBITS
    cores = os.cpu_count() or 1
    scratch = default_scratch()
    if not ref_store_ok(scratch, n):
        return {"impl": "reference", "unavailable": f"{scratch} has < 17.6 GB free for the n=30 reference store"}
    ops = sweep_ops()
    order = stratified_order()
    walls = []
    with eng.store(n, 65536, 0, scratch) as store:
        for k in range(args.warmup):
            store.apply(ops[[order[(len(order) - args.warmup + k) % len(order)]]], "paired-cached-parallel", cores,
                        cores * (64 << 20))
        for k in range(args.steps):
            walls.append(store.apply(ops[[order[k % len(order)]]], "paired-cached-parallel", cores,
                                     cores * (64 << 20)))
    ms = sum(walls) / len(walls)
    value = (1 << n) / (ms / 1e3)
    sample = (f"{args.steps} steps of 1 sweep gate each (order U0,CX,CX,CX,U1,...: the sweep's 1:3 mix"
              f"{' exactly' if args.steps % 4 == 0 else ''}), reference apply_circuit paired-cached-parallel, "
              f"workers={cores}, block_amps=65536, store on {scratch}; Metrics.wall_ms per step; the CPU runs "
              f"the n=30 sweep (2^30 amplitudes, the per-GPU shard size) at every N")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded Haar-random unitaries, mt19937_64 seed 2508; committed gate records)",
            "config": bench_config(n + int(math.log2(world)), n, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def config4_leg(qv, line, args, rank, world, dist):
    """BASELINE config 4 (weak scaling): the U3 + CX-ladder layer circuit (20
    layers) at n = 32 + log2 N, a 64 GiB complex128 shard per GPU, through the
    API defaults (fused passes; global-qubit gates trigger exchanges over
    peer memory / NCCL). value = ops * 2^n / t_step (whole job), CUDA events on
    the state's stream, max over ranks. At N > 1 the engine times every
    local-pass batch and exchange (QVG_OPT_TIMING)."""
    import torch

    g = int(math.log2(world))
    n = 32 + g
    dev = torch.cuda.current_device()
    free, _ = torch.cuda.mem_get_info(dev)
    if free < (16 << (n - g)) * 1.05:
        line["config4"] = {"skipped": f"needs {(16 << (n - g)) / 2**30:.0f} GiB free, {free / 2**30:.0f} GiB free"}
        return
    c = qv.u3_ladder_circuit(n, 20, 1)
    if world == 1:
        st = qv.StateVector.create(n, 128, dev)
    else:
        box = [qv.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        st = qv.StateVector.create_sharded(n, 128, dev, rank, world, box[0])
        st.set_option(qv.OPT_TIMING, 1)
    stream = torch.cuda.ExternalStream(st.stream(), device=dev)
    qv.apply_circuit(st, c)  # warm-up (plans, exchange mappings)
    st.sync()
    st.reset_stats()
    steps = max(1, min(args.steps, 3))
    if dist is not None:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        qv.apply_circuit(st, c, sync=False)
    b.record(stream)
    st.sync()
    ms = a.elapsed_time(b) / steps
    s = st.stats()
    vals = [ms, s["kernel_ms"] / steps, s["exchange_ms"] / steps, s["exchange_bytes"] / steps]
    if dist is not None:
        t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = [float(v) for v in t.tolist()]
    ms, k_ms, x_ms, x_bytes = vals
    out = {"workload": f"config4: U3 layers + CX ladder, 20 layers, n={n} ({world} x 64 GiB c128 shards), "
                       "API defaults (fused, exchanges)",
           "value": len(c) * (1 << n) / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
           "ops": len(c), "passes_per_step": s["passes"] / steps, "exchanges_per_step": s["exchanges"] / steps,
           "hbm_gbs_per_gpu": s["bytes_moved"] / steps / (ms / 1e3) / 1e9,
           "timing": "CUDA events on the state's stream around the steps (the circuit applied again to the "
                     "evolving state each step), max over ranks"}
    if world > 1:
        out["exchange"] = {"bytes_per_step_per_gpu": x_bytes, "ms_per_step": x_ms,
                           "gbs_per_gpu": x_bytes / (x_ms / 1e3) / 1e9 if x_ms else None, "peak_gbs": 900.0,
                           "frac": x_bytes / (x_ms / 1e3) / 1e9 / 900.0 if x_ms else None,
                           "local_pass_ms_per_step": k_ms}
    line["config4"] = out
    del st


def configs_mode(args):
    """`--configs`: one JSON line per BASELINE config with device
    time fused (API default) and per-gate, HBM passes, amp-updates/s, and the
    reference engine (oracle/_ref, all host cores) on the same circuit or a
    bounded sample of it (stated in each line). Not the driver's headline."""
    import torch

    from oracle.oracle import GATE_DTYPE, RefEngine, default_scratch

    import paper_2508_15545_b200 as qv

    cores = os.cpu_count() or 1
    eng = RefEngine() if RefEngine.available() else None
    specs = [
        ("config0", "U3 layers + CX ladder, n=20, 20 layers", lambda: qv.u3_ladder_circuit(20, 20, 1), 128, None),
        ("config1", "H layer + QFT (CP R_k) + bit-reversal SWAPs, n=26, seeded basis input",
         lambda: qv.qft_circuit(26, 1)[0], 128, 60),
        ("config2_c128", "Haar U on q=0..29 + 90 CX, n=30", lambda: qv.haar_sweep_circuit(30, SEED), 128, 2),
        ("config2_c64", "Haar U on q=0..29 + 90 CX, n=30, complex64", lambda: qv.haar_sweep_circuit(30, SEED), 64, 2),
        ("config3", "5x6 grid, 24 cycles of sqrt-X/Y/W + CZ patterns, n=30", lambda: qv.grid_circuit(5, 6, 24, 1),
         128, 2),
        ("config4_g1", "U3 layers + CX ladder, n=32 on 1 GPU (64 GiB), 20 layers",
         lambda: qv.u3_ladder_circuit(32, 20, 1), 128, 0),
    ]
    for name, desc, build, prec, sample in specs:
        c = build()
        n = c.n_qubits
        g = c.gates()
        st = qv.StateVector.create(n, prec, 0)
        stream = torch.cuda.ExternalStream(st.stream())
        res = {}
        for mode, fuse in (("fused", 1), ("per_gate", 0)):
            st.set_option(qv.OPT_FUSE, fuse)
            st.apply_gates(g)  # warm-up
            st.reset_stats()
            reps = 1 if n >= 32 else 5  # median of reps (small states are launch-bound and noisy)
            times = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.apply_gates(g, sync=False)
                e1.record(stream)
                st.sync()
                times.append(e0.elapsed_time(e1))
            ms = sorted(times)[len(times) // 2]
            s = st.stats()
            res[mode] = {"ms": ms, "reps": reps, "passes": s["passes"] // reps,
                         "amp_updates_per_s": len(c) * (1 << n) / (ms / 1e3),
                         "hbm_gbs": s["bytes_moved"] / reps / (ms / 1e3) / 1e9}
        del st
        cpu = None
        if eng is not None and sample != 0:
            ops = np.frombuffer(g.tobytes(), dtype=GATE_DTYPE)
            part = ops if sample is None else ops[:sample]
            with eng.store(n, 65536, 0, default_scratch()) as rs:
                wall = rs.apply(part, "paired-cached-parallel", cores, cores * (64 << 20))
            per_gate = wall / len(part)
            cpu = {"ms_total" if sample is None else "ms_total_extrapolated": per_gate * len(c),
                   "ms_per_gate": per_gate, "cores": cores, "kind": "reference",
                   "sample": "whole circuit" if sample is None else f"first {len(part)} ops"}
        elif sample == 0:
            cpu = {"note": "n=32 state is 64 GiB: reference CPU run infeasible here; "
                           "extrapolate x4 per gate from config2 (SPEC.md:618 growth law)"}
        print(json.dumps({"config": name, "workload": desc, "n_qubits": n, "precision": prec, "ops": len(c),
                          "gpu": res, "speedup_fused_vs_per_gate": res["per_gate"]["ms"] / res["fused"]["ms"],
                          "cpu_reference": cpu}), flush=True)


def relaunch_or_fail(args):
    """--gpus N > 1 without torchrun: re-launch under torch.distributed.run
    with N ranks when N GPUs are visible; otherwise fail loudly (a one-GPU run
    must never print n_gpus: 1 for --gpus N)."""
    try:
        import torch

        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but {have} CUDA device(s) visible"}), flush=True)
        sys.exit(2)
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"))
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-config4", action="store_true")
    ap.add_argument("--configs", action="store_true", help="per-config lines (C0..C4) instead of the headline")
    args = ap.parse_args()
    if args.configs:
        configs_mode(args)
        return
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    if args.gpus < 1 or args.gpus & (args.gpus - 1):
        ap.error("--gpus must be a power of two")
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1 and args.impl == "ours":
        relaunch_or_fail(args)
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus and args.impl == "ours":
        print(json.dumps({"error": f"WORLD_SIZE={world} but --gpus {args.gpus}"}), flush=True)
        sys.exit(2)
    dist = None
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist

        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the communicator lines show the N ranks
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        tdist.init_process_group("nccl")
        dist = tdist
    import paper_2508_15545_b200 as qv

    st, circ, recs, line, n = run_ours(args, rank, world, dist)
    if world == 1:
        fused_leg(qv, st, circ, line, args)
        if not args.no_e2e:
            e2e_leg(qv, st, circ, recs, line, args)
        c64_leg(qv, circ, recs, line, args)
    elif not args.no_e2e:
        e2e_leg_sharded(qv, st, circ, line, args, rank, world, dist)
    del st
    if not args.no_config4:
        try:
            config4_leg(qv, line, args, rank, world, dist)
        except Exception as exc:  # keep the headline line if the 64 GiB leg cannot run
            line["config4"] = {"error": str(exc)[:200]}
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(args)
            except Exception as exc:  # keep the GPU line even if the host run fails
                line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
