"""QVSV state files: our StateStore and the reference's BlockStore read and
write the same bytes (reference store.hpp:24-29, store.cpp:181-316), so the
file-backed `apply_circuit(store, circuit, strategy="gpu")` is a drop-in for
the reference's strategies on the same file."""
import os
import shutil

import numpy as np
import pytest

from conftest import gate_array
from oracle.oracle import RefEngine

needs_ref = pytest.mark.skipif(not RefEngine.available(), reason="oracle/_ref not built")


def test_create_matches_reference_bytes(qv, tmp_path):
    # |0...0> stores from both implementations are byte-identical
    ours = tmp_path / "ours.qvs"
    s = qv.StateStore.create(str(ours), 6, block_amps=4)
    assert (s.n_qubits, s.n_amps, s.block_amps, s.n_blocks) == (6, 64, 4, 16)
    assert s.path == str(ours)
    del s
    raw = ours.read_bytes()
    assert raw[:4] == b"QVSV" and len(raw) == 32 + 64 * 16
    assert int.from_bytes(raw[4:8], "little") == 1 and int.from_bytes(raw[8:12], "little") == 6
    assert int.from_bytes(raw[12:20], "little") == 4 and raw[20:32] == bytes(12)
    amps = np.frombuffer(raw[32:], np.complex128)
    assert amps[0] == 1 and not amps[1:].any()
    if RefEngine.available():
        eng = RefEngine()
        with eng.store(6, block_amps=4, scratch=str(tmp_path)) as ref:
            ref.sync()
            ref_bytes = None
            for f in tmp_path.iterdir():
                if f.name.startswith("qvr-"):
                    ref_bytes = f.read_bytes()
        assert ref_bytes == raw


@needs_ref
def test_reference_file_readable_and_ours_readable_by_reference(qv, tmp_path):
    eng = RefEngine()
    ops, _ = eng.random_circuit(8, 60, 4)
    path = str(tmp_path / "a.qvs")
    qv.StateStore.create(path, 8, block_amps=16)
    ref = eng.open_store(path, 8)
    ref.apply(ops, "paired-cached", 1, 4 * 16 * 16)
    want = ref.read()
    ref_norm = ref.norm()
    ref.close()
    s = qv.StateStore.open(path)
    assert np.array_equal(s.read_state(), want)
    assert s.norm() == ref_norm  # same Kahan order
    assert s.amplitude(5) == want[5]
    p = np.abs(want) ** 2
    order = sorted(range(len(p)), key=lambda i: (-p[i], i))[:6]
    assert [i for i, _ in qv.top_amplitudes(s, 6)] == order


def test_bad_files(qv, tmp_path):
    p = tmp_path / "bad.qvs"
    p.write_bytes(b"QVSX" + bytes(28) + bytes(64))
    with pytest.raises(qv.FormatError):
        qv.StateStore.open(str(p))
    p.write_bytes(b"QV")
    with pytest.raises(qv.FormatError):
        qv.StateStore.open(str(p))
    good = tmp_path / "g.qvs"
    qv.StateStore.create(str(good), 3)
    data = good.read_bytes()
    good.write_bytes(data[:-16])
    with pytest.raises(qv.FormatError, match="length"):
        qv.StateStore.open(str(good))
    with pytest.raises(qv.IoError):
        qv.StateStore.create(str(good), 3)  # exists, no overwrite
    with pytest.raises(qv.ValidationError):
        qv.StateStore.create(str(tmp_path / "x.qvs"), 4, block_amps=3)
    with pytest.raises(qv.ValidationError):
        qv.apply_circuit(qv.StateStore.create(str(tmp_path / "y.qvs"), 3), qv.parse_circuit("qubits 3\nh 0\n"),
                         strategy="paired-cached")


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("n", [10, 22])
def test_gpu_strategy_on_store_matches_reference_strategy(qv, tmp_path, n):
    """Same file, reference `paired-cached-parallel` vs our `gpu`."""
    eng = RefEngine()
    c = qv.u3_ladder_circuit(n, 3, 9)
    a = str(tmp_path / "a.qvs")
    qv.StateStore.create(a, n, block_amps=1024)
    b = str(tmp_path / "b.qvs")
    shutil.copyfile(a, b)
    ref = eng.open_store(a, n)
    ref.apply(gate_array(c), "paired-cached-parallel", 4, 4 * (64 << 20))
    want = ref.read()
    ref.close()
    m = qv.apply_circuit(qv.StateStore.open(b), c, strategy="gpu")
    assert m["strategy"] == "gpu" and m["gates_applied"] == len(c)
    assert m["bytes_read"] == m["bytes_written"] == 16 << n
    # the reference's normative metrics fields (reference metrics.cpp:25-41)
    for key in ("n_qubits", "strategy", "workers", "gates_applied", "traversals", "blocks_read", "blocks_written",
                "bytes_read", "bytes_written", "cache_hits", "cache_misses", "peak_cache_bytes", "wall_ms"):
        assert key in m, key
    assert m["blocks_read"] == m["blocks_written"] == (1 << n) // min(1024, 1 << n)
    assert m["peak_cache_bytes"] >= 16 << n
    got = qv.StateStore.open(b).read_state()
    assert np.array_equal(got, want)
    # and the reference can continue on our output
    ref = eng.open_store(b, n)
    assert np.array_equal(ref.read(), want)
    ref.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n,w", [(16, 8), (20, 12), (22, 14)])
def test_store_streamed_through_hbm_windows_matches_resident(qv, tmp_path, n, w):
    """Out-of-core from a file: the state streams through
    two 2^w-amplitude HBM windows segment by segment; the result is bit-exact
    with the whole-state-resident apply of the same circuit on the same file."""
    c = qv.random_circuit(n, 400, 7)
    a = str(tmp_path / "a.qvs")
    qv.StateStore.create(a, n, block_amps=256)
    b = str(tmp_path / "b.qvs")
    shutil.copyfile(a, b)
    m_res = qv.apply_circuit(qv.StateStore.open(a), c, strategy="gpu")
    m_str = qv.apply_circuit(qv.StateStore.open(b), c, strategy="gpu", window_qubits=w)
    assert m_str["gates_applied"] == m_res["gates_applied"] == len(c)
    assert m_str["exchanges"] >= 2  # random targets over all n qubits need >1 segment
    assert m_str["bytes_read"] == m_str["bytes_written"] == m_str["exchanges"] * (16 << n)
    want = qv.StateStore.open(a).read_state()
    got = qv.StateStore.open(b).read_state()
    assert np.array_equal(got, want)
    if n <= 16:
        from oracle.oracle import Oracle
        o = Oracle()
        ops, _ = o.random_circuit(n, 400, 7)
        init = np.zeros(1 << n, np.complex128)
        init[0] = 1
        assert np.array_equal(o.apply(n, init, ops), got)


@pytest.mark.gpu
def test_reference_positional_signature(qv, tmp_path):
    """apply_circuit(store, circuit, strategy, cache_bytes, workers) as the
    reference binding orders it (reference bindings/module.cpp:118-139)."""
    path = str(tmp_path / "p.qvs")
    qv.StateStore.create(path, 12, block_amps=64)
    c = qv.random_circuit(12, 100, 3)
    m = qv.apply_circuit(qv.StateStore.open(path), c, "gpu", 64 << 20, 4)
    assert m["gates_applied"] == 100
    with pytest.raises(qv.ValidationError):
        qv.apply_circuit(qv.StateStore.open(path), c, "gpu", 64 << 20, 0)
    with pytest.raises(qv.ValidationError, match="paired-cached"):
        qv.apply_circuit(qv.StateStore.open(path), c, "paired-cached")


def _header(magic=b"QVSV", version=1, n=4, block_amps=4, reserved=bytes(12)):
    return (magic + version.to_bytes(4, "little") + n.to_bytes(4, "little") + block_amps.to_bytes(8, "little")
            + reserved)


FILES = {
    "good": _header() + bytes(16 * 16),
    "bad_magic": _header(magic=b"QVSX") + bytes(16 * 16),
    "version_2": _header(version=2) + bytes(16 * 16),
    "version_0": _header(version=0) + bytes(16 * 16),
    "n_zero": _header(n=0) + bytes(16),
    "n_huge": _header(n=60) + bytes(16),
    "block_not_pow2": _header(block_amps=3) + bytes(16 * 16),
    "block_zero": _header(block_amps=0) + bytes(16 * 16),
    "block_over_state": _header(block_amps=32) + bytes(16 * 16),
    "truncated_payload": _header() + bytes(16 * 15),
    "extra_payload": _header() + bytes(16 * 17),
    "short_header": b"QVSV" + bytes(20),
    "empty": b"",
    "reserved_nonzero": _header(reserved=b"\x01" + bytes(11)) + bytes(16 * 16),
}


@needs_ref
@pytest.mark.parametrize("name", sorted(FILES))
def test_open_errors_match_reference(qv, tmp_path, name):
    """StateStore.open accepts exactly the files the reference's
    BlockStore::open accepts, with the same error class
    (reference store.cpp:135-149,216-245; tests/test_store.cpp:78-95,142-154)."""
    p = tmp_path / f"{name}.qvs"
    p.write_bytes(FILES[name])
    want = RefEngine().open_error(str(p))
    try:
        qv.StateStore.open(str(p))
        got = None
    except qv.QvsimError as e:
        got = type(e).__name__
    assert got == want, (name, got, want)
