"""BASELINE configs 2, 3 and 4 at their stated sizes (VERDICT r1 "missing" #1).

* Configs 2 and 3 (n = 30, complex128): the GPU state must hash, chunk by
  chunk, to the UNMODIFIED reference engine's final state
  (tests/golden/ref_full.json, generated once by
  tests/golden/make_golden_full.py through oracle/_ref); norm, top-8 and 1024
  seeded sample amplitudes are compared too. Fused (API default) and one pass
  per gate.
* Config 2 in complex64: max |delta| <= 1e-5 against the complex128 GPU state
  whose hashes matched the reference, fidelity >= 1 - 1e-10 is for
  complex128 (bit-identical here).
* Config 4 (n = 32, 33; 64 / 128 GiB on one B200): the reference cannot run
  it, so the worker-count law stands in
  (reference tests/acceptance.cpp:196-242): the unsharded run and 2 / 4 / 8
  virtual shards (the multi-GPU schedule, exchanges and batched exchanges on
  one device) must hash identically, and the norm drift stays <= 1e-10
  (reference tests/acceptance.cpp:398-419).
"""
import hashlib
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import ROOT, gate_array

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden")
CHUNK = 1 << 26


def fixture(name):
    path = os.path.join(GOLD, "ref_full.json")
    with open(path) as f:
        fx = json.load(f)
    if name not in fx:
        pytest.fail(f"fixture {name} missing from {path}: run tests/golden/make_golden_full.py")
    return fx[name]


def chunk_hashes(st, chunk=CHUNK):
    """sha256 of every `chunk`-amplitude slice of the state (complex128 host
    bytes), D2H of the next chunk overlapping the hashing of the previous."""
    total = 1 << st.n_qubits
    out, futs = [], []
    with ThreadPoolExecutor(6) as pool:
        for o in range(0, total, chunk):
            if len(futs) >= 6:  # bound the host memory held by chunks in flight
                out.append(futs.pop(0).result())
            a = st.read_state(o, min(chunk, total - o))
            futs.append(pool.submit(lambda a: hashlib.sha256(a.data).hexdigest(), a))
        out += [f.result() for f in futs]
    return out


def circuit_of(qv, fx):
    out = getattr(qv, fx["builder"])(*fx["args"])
    c = out[0] if isinstance(out, tuple) else out
    ops = gate_array(c)
    assert hashlib.sha256(ops.tobytes()).hexdigest() == fx["ops_sha256"]  # the builder still emits these bytes
    saved = np.load(os.path.join(GOLD, fx["ops_file"]))
    assert saved.tobytes() == ops.tobytes()
    return c


def check_against_reference(qv, st, fx):
    assert chunk_hashes(st, fx["chunk_amps"]) == fx["chunk_sha256"]
    assert abs(st.norm() - fx["norm"]) <= 1e-13
    top = st.top_amplitudes(8)
    assert [i for i, _ in top] == fx["top8_index"]
    assert all(v == complex(*w) for (_, v), w in zip(top, fx["top8"]))
    idx = np.sort(np.random.default_rng(fx["sample_seed"]).choice(1 << fx["n_qubits"], len(fx["samples"]),
                                                                   replace=False))
    want = np.array([complex(*w) for w in fx["samples"]])
    got = np.array([st.amplitude(int(i)) for i in idx])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", ["config2_haar_sweep_n30", "config3_grid_5x6_c24_n30"])
def test_n30_configs_match_reference_engine(qv, name):
    fx = fixture(name)
    c = circuit_of(qv, fx)
    for fuse in (True, False):
        st = qv.StateVector.create(30, 128, 0)
        m = qv.apply_circuit(st, c, fuse=fuse)
        assert m["traversals"] < len(c) if fuse else m["traversals"] <= len(c)
        check_against_reference(qv, st, fx)
        del st


def test_config2_n30_complex64_within_tolerance(qv):
    """c64 against the c128 GPU state (bit-identical to the reference, checked
    by hash first): max |delta| <= 1e-5 (north_star), per gate and fused."""
    fx = fixture("config2_haar_sweep_n30")
    c = circuit_of(qv, fx)
    ref = qv.StateVector.create(30, 128, 0)
    qv.apply_circuit(ref, c)
    assert chunk_hashes(ref) == fx["chunk_sha256"]
    for fuse in (True, False):
        st = qv.StateVector.create(30, 64, 0)
        qv.apply_circuit(st, c, fuse=fuse)
        worst = 0.0
        for off in range(0, 1 << 30, CHUNK):
            worst = max(worst, float(np.abs(st.read_state(off, CHUNK) - ref.read_state(off, CHUNK)).max()))
        assert worst <= 1e-5, (fuse, worst)
        assert abs(st.norm() - 1.0) <= 1e-5
        del st


def _free_gib(qv):
    import torch

    free, _ = torch.cuda.mem_get_info(0)
    return free / 2**30


@pytest.mark.parametrize("n", [32, 33])
def test_config4_worker_count_law_full_size(qv, n):
    """Config 4 (U3 + CX ladder, 20 layers) at n = 32 and 33: the unsharded
    state and 2 / 4 / 8 virtual shards have identical device chunk checksums
    (qvg_checksums, 2 x 64 bits per 2^26 amplitudes, every bit including the
    sign of zeros; checked against host sha256 for the unsharded n = 32 run),
    and the norm drift is <= 1e-10."""
    need = (16 << n) / 2**30 * 1.05
    if _free_gib(qv) < need:
        pytest.fail(f"n={n} needs {need:.0f} GiB of HBM")
    c = qv.u3_ladder_circuit(n, 20, 1)
    hashes = {}
    for world in (1, 2, 4, 8):
        st = (qv.StateVector.create(n, 128, 0) if world == 1
              else qv.StateVector.create_sharded(n, 128, 0, 0, world, None))
        m = qv.apply_circuit(st, c)
        if world > 1:
            assert m["exchanges"] > 0
        assert abs(st.norm() - 1.0) <= 1e-10
        hashes[world] = st.checksums(CHUNK)
        if world == 1 and n == 32:  # the device words agree with the host's view of the bytes
            from conftest import checksums_numpy

            for k in (0, 17, 63):
                assert np.array_equal(checksums_numpy(st.read_state(k * CHUNK, CHUNK), CHUNK, k * CHUNK)[0],
                                      hashes[1][k])
        del st
    for world in (2, 4, 8):
        assert np.array_equal(hashes[world], hashes[1]), world


def test_topk_n32_uniform_state_64bit_bins(qv):
    """2^32 equal keys fall in one radix bin (a 32-bit histogram wraps to 0,
    ADVICE r1): the top-3 of the uniform n=32 state are indices 0, 1, 2."""
    if _free_gib(qv) < 66:
        pytest.fail("n=32 needs 64 GiB of HBM")
    st = qv.StateVector.create(32, 128, 0)
    qv.apply_circuit(st, qv.make_benchmark_circuit(32))
    top = st.top_amplitudes(3)
    assert [i for i, _ in top] == [0, 1, 2]
    assert all(abs(v - 2.0 ** -16) <= 1e-18 for _, v in top)
