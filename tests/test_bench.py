"""bench.py's contract pieces that run without a GPU: the reference arm's
inputs (committed gate records, pinned to the package's builder), its
stratified one-gate steps, and the --gpus guard."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

from conftest import ROOT, gate_array

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_sweep_records_match_builder(qv):
    """The reference arm loads the sweep from tests/golden (no package import);
    those bytes are exactly what haar_sweep_circuit(30, 2508) emits."""
    ops = bench.sweep_ops()
    assert len(ops) == 120
    assert ops.tobytes() == gate_array(qv.haar_sweep_circuit(30, bench.SEED)).tobytes()
    with open(bench.SWEEP_FIXTURE) as f:
        assert json.load(f)["config2_haar_sweep_n30"]["ops_sha256"] == hashlib.sha256(ops.tobytes()).hexdigest()


def test_stratified_order_keeps_the_mix():
    order = bench.stratified_order()
    assert sorted(order) == list(range(120))  # a cycle is the whole sweep once
    ops = bench.sweep_ops()
    kinds = ops["kind"][order]
    for k in range(0, 120, 4):
        assert list(kinds[k:k + 4]) == [0, 1, 1, 1]


def test_reference_arm_does_not_import_the_package():
    src = open(os.path.join(ROOT, "bench.py")).read()
    body = src[src.index("def run_reference("):src.index("def config4_leg(")]
    assert "paper_2508_15545_b200" not in body and "import qv" not in body
    body = src[src.index("def cpu_baseline("):src.index("def run_reference(")]
    assert "paper_2508_15545_b200" not in body


def test_gpus_flag_fails_without_enough_devices():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env)
    import torch

    if torch.cuda.device_count() < 2:
        assert r.returncode == 2 and "requested" in r.stdout
    env["WORLD_SIZE"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stdout


def test_granule_bytes():
    ops = bench.sweep_ops()
    raw = np.frombuffer(ops.tobytes(), np.uint8).reshape(-1, 80)
    total = (1 << 30) * 16
    for rec, op in zip(raw, ops):
        g, a = bench.granule_bytes(30, rec), bench.algorithmic_bytes(30, rec)
        if op["kind"] == 0:
            assert g == a == 2 * total
        elif op["control"] in (1, 2):  # 32 / 64-B control runs: whole state read, half written
            assert g == total + total // 2 and a == total
        elif op["control"] == 0:  # 16-B runs: everything moves
            assert g == 2 * total
        else:
            assert g == a == total
