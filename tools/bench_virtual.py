"""bench.py's N > 1 step (the whole sweep per call, sharded state, exchange
schedule, apportioned per-gate times, exchange roofline) on ONE device with
virtual shards, so the multi-GPU bookkeeping runs on hardware without
several GPUs (no NCCL, no ranks waiting on each other).

    python tools/bench_virtual.py [--world 2] [--steps 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    _, _, _, line, _ = bench.run_ours(argparse.Namespace(steps=a.steps, warmup=a.warmup), 0, a.world, None)
    keep = ("value", "ms_per_step", "n_gpus", "config", "roofline", "exchanges_per_step", "exchange_roofline",
            "gpu_launches", "per_gate_timing")
    print(json.dumps({k: line[k] for k in keep if k in line}))


if __name__ == "__main__":
    main()
