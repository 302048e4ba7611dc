"""Host-side logic on CPU: the C++ host mirror of the reference API (circuit
text, seeded generator, config builders), the pass planner, and the C-ABI
library's exports. No device work."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, gate_array
from oracle.oracle import GATE_DTYPE

GOLD = os.path.join(ROOT, "tests", "golden")


def cuda_present():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


# --- reference API parity ---------------------------------------------------------
def test_random_circuit_matches_reference(qv):
    gold = np.load(os.path.join(GOLD, "ref_random.npz"))
    for key in sorted({k.rsplit("_", 1)[0] for k in gold.files}):
        n, d, s = (int(x[1:]) for x in key.split("_"))
        c = qv.random_circuit(n, d, s)
        assert c.gates().tobytes() == gold[f"{key}_ops"].tobytes(), key
        assert c.to_text() == gold[f"{key}_text"].tobytes().decode(), key


def test_text_round_trip_and_determinism(qv):
    # reference tests/python/test_smoke.py:28-44
    c = qv.random_circuit(5, 25, 42)
    text = c.to_text()
    back = qv.parse_circuit(text)
    assert back.n_qubits == 5 and len(back) == 25
    assert back.to_text() == text == qv.serialize_circuit(back)
    assert qv.random_circuit(4, 30, 7).to_text() == qv.random_circuit(4, 30, 7).to_text()
    assert qv.random_circuit(4, 30, 7).to_text() != qv.random_circuit(4, 30, 8).to_text()


def test_extended_grammar_round_trips(qv):
    text = "qubits 4\ncp 0 3 0.39269908169872414\ncu 1 2 0 0 1 0 1 0 0 0\np 2 1.5\nu3 1 0.5 0.25 0.125\nsx 0\nsy 1\nsw 2\ncx 3 0\ncz 1 0\n"
    c = qv.parse_circuit(text)
    assert c.to_text() == text
    assert qv.parse_circuit(c.to_text()).gates().tobytes() == c.gates().tobytes()


def test_swap_instruction_and_config_round_trips(qv):
    """`swap a b` expands to cx a b / cx b a / cx a b (config 1's bit
    reversal); every BASELINE config builder round-trips as text bit for bit
    (SURVEY §8f row 4)."""
    c = qv.parse_circuit("qubits 5\nswap 1 4\n")
    assert c.to_text() == "qubits 5\ncx 1 4\ncx 4 1\ncx 1 4\n"
    with pytest.raises(qv.ParseError, match="itself"):
        qv.parse_circuit("qubits 3\nswap 2 2\n")
    with pytest.raises(qv.ParseError, match="line 2"):
        qv.parse_circuit("qubits 3\nswap 0 7\n")
    for c in [qv.u3_ladder_circuit(20, 20, 1), qv.qft_circuit(26, 1)[0], qv.haar_sweep_circuit(30, 2508),
              qv.grid_circuit(5, 6, 24, 1), qv.u3_ladder_circuit(35, 20, 4)]:
        back = qv.parse_circuit(c.to_text())
        assert back.gates().tobytes() == c.gates().tobytes()


def test_errors_are_typed_with_lines(qv):
    # reference tests/python/test_smoke.py:110-123
    with pytest.raises(qv.QvsimError, match="line 2"):
        qv.parse_circuit("qubits 2\nh 7\n")
    with pytest.raises(qv.ParseError):
        qv.parse_circuit("h 0\n")
    with pytest.raises(qv.ParseError, match="unknown instruction"):
        qv.parse_circuit("qubits 2\nfoo 0\n")
    with pytest.raises(qv.ParseError, match="control equals target"):
        qv.parse_circuit("qubits 2\ncx 1 1\n")
    with pytest.raises(qv.ParseError, match="not unitary"):
        qv.parse_circuit("qubits 1\nu 0 1 0 1 0 0 0 1 0\n")


def test_gate_library(qv):
    r = 1 / math.sqrt(2)
    assert np.allclose(qv.make_gate("h"), [r, r, r, -r])
    sx = np.array(qv.make_gate("sx")).reshape(2, 2)
    assert np.allclose(sx @ sx, [[0, 1], [1, 0]], atol=1e-15)
    sy = np.array(qv.make_gate("sy")).reshape(2, 2)
    assert np.allclose(sy @ sy, [[0, -1j], [1j, 0]], atol=1e-15)
    sw = np.array(qv.make_gate("sw")).reshape(2, 2)
    w = np.array([[0, (1 - 1j) * r], [(1 + 1j) * r, 0]])
    assert np.allclose(sw @ sw, w, atol=1e-15)
    th, ph, la = 0.3, 1.1, 2.5
    u3 = np.array(qv.make_gate("u3", [th, ph, la])).reshape(2, 2)
    want = np.array([[math.cos(th / 2), -np.exp(1j * la) * math.sin(th / 2)],
                     [np.exp(1j * ph) * math.sin(th / 2), np.exp(1j * (ph + la)) * math.cos(th / 2)]])
    assert np.allclose(u3, want, atol=1e-15)


# --- BASELINE config builders -------------------------------------------
def test_config_builders_shapes(qv):
    c0 = qv.u3_ladder_circuit(20, 20, 1)
    assert len(c0) == 20 * (20 + 19)
    c1, b = qv.qft_circuit(26, 1)
    names = c1.names()
    assert names.count("cp") == 325 and names.count("h") == 52 and names.count("cx") == 39
    assert names.count("x") == bin(b).count("1") and 0 <= b < 2 ** 26
    c2 = qv.haar_sweep_circuit(30, 2508)
    assert c2.names().count("u") == 30 and c2.names().count("cx") == 90
    c3 = qv.grid_circuit(5, 6, 24, 1)
    nm = c3.names()
    assert sum(nm.count(g) for g in ("sx", "sy", "sw")) == 720 and nm.count("cz") == 294
    # never the same 1q gate twice in a row on a qubit
    ops = gate_array(c3)
    last = {}
    for name, op in zip(nm, ops):
        if name in ("sx", "sy", "sw"):
            assert last.get(int(op["target"])) != name
            last[int(op["target"])] = name


def test_haar_unitaries(qv):
    ops = gate_array(qv.haar_sweep_circuit(30, 2508))[:30]
    for op in ops:
        u = op["u"].view(np.complex128).reshape(2, 2)
        assert np.abs(u.conj().T @ u - np.eye(2)).max() < 1e-14


# --- planner -------------------------------------------------------------------------
def test_planner_bytes_and_fusion(qv):
    n, S = 20, 16
    full = 2 * (1 << n) * S
    one = lambda text: qv.plan_passes(n, qv.parse_circuit(f"qubits {n}\n{text}\n").gates(), fuse=False)
    assert one("h 7") == (1, 0, full)
    assert one("cx 3 9") == (1, 0, full // 2)       # only control=1 amplitudes
    assert one("cx 0 9") == (1, 0, full)           # control bit 0: sector-rounded
    assert one("cz 4 9") == (1, 0, full // 4)       # diag(1,-1) with control: |11> quarter
    assert one("t 9") == (1, 0, full // 2)
    assert one("cp 2 9 0") == (0, 0, 0)            # identity: no pass
    # 11 Hadamards on 0..10 fuse into one tile pass (default tile: 11 qubits);
    # a 12th target needs a second pass
    text = "\n".join(f"h {q}" for q in range(11))
    assert qv.plan_passes(n, qv.parse_circuit(f"qubits {n}\n{text}\n").gates()) == (1, 1, full)
    text += "\nh 11"
    assert qv.plan_passes(n, qv.parse_circuit(f"qubits {n}\n{text}\n").gates())[:2] == (2, 1)
    assert qv.plan_passes(n, qv.parse_circuit(f"qubits {n}\n{text}\n").gates(), tile_qubits=12) == (1, 1, full)
    # config 3 (n=30): fused passes are far fewer than ops
    c3 = qv.grid_circuit(5, 6, 24, 1)
    p, f, b = qv.plan_passes(30, c3.gates())
    assert f == p and p < len(c3) / 8


def test_planner_uses_engine_shape(qv):
    """plan_passes plans with the engine's own defaults: complex64
    tiles are 12 qubits, complex128 11, and complex128 states of <= 17 qubits
    use 10-qubit tiles unless the caller picks a shape."""
    h = lambda n, k: qv.parse_circuit(f"qubits {n}\n" + "\n".join(f"h {q}" for q in range(k)) + "\n").gates()
    assert qv.plan_passes(20, h(20, 12), precision=64)[:2] == (1, 1)
    assert qv.plan_passes(20, h(20, 12), precision=128)[:2] == (2, 1)
    assert qv.plan_passes(16, h(16, 11))[:2] == (2, 1)                    # small state: 10-qubit tiles
    assert qv.plan_passes(16, h(16, 11), tile_qubits=11)[:2] == (1, 1)    # caller's shape wins
    assert qv.plan_passes(18, h(18, 11))[:2] == (1, 1)


def test_planner_bit_exact_reorder(qv):
    # The default plan lets X/CX permutations and Z/CZ sign flips move past
    # ops on other qubits (bit-exact, qvg_plan.hpp reorder_for_tiles); the
    # U3 + CX ladder then needs about half the passes of circuit order
    # (27 at n=30, 4 layers).
    p, f, _ = qv.plan_passes(30, qv.u3_ladder_circuit(30, 4, 1).gates())
    assert f == p and p == 14


@pytest.mark.parametrize("prec,S", [(128, 16), (64, 8)])
def test_counter_law_per_gate_plan(qv, oracle, prec, S):
    """The reference's single-traversal law (SPEC.md:393,
    proj/tests/test_kernel.cpp:253-277: one traversal per gate, an exact
    equality) for the per-gate plan: passes = non-identity ops, and the
    planner's bytes equal SURVEY §8d's per-gate bytes summed over the ops,
    computed here from the table alone."""
    from conftest import algorithmic_bytes
    for n, depth, seed in ((6, 200, 1), (12, 300, 2), (20, 300, 3), (30, 200, 4)):
        ops, _ = oracle.random_circuit(n, depth, seed)
        want = [algorithmic_bytes(n, S, op) for op in ops]
        p, f, b = qv.plan_passes(n, ops.tobytes(), precision=prec, fuse=False)
        assert f == 0 and p == sum(1 for w in want if w) and b == sum(want)
        for op, w in list(zip(ops, want))[:40]:  # and gate by gate
            assert qv.plan_passes(n, op.tobytes(), precision=prec, fuse=False) == (1 if w else 0, 0, w)


def test_counter_law_fused_plan(qv, oracle):
    """A fused pass costs one traversal of the state whatever it holds
    (SURVEY §8d): a plan's bytes are its fused passes * 2 * 2^n * S plus the
    per-gate bytes of the ops left unfused, and never more than one pass per
    gate would cost in traversals."""
    for n, depth, seed in ((14, 400, 5), (24, 600, 6), (30, 800, 7)):
        ops, _ = oracle.random_circuit(n, depth, seed)
        full = 2 * (1 << n) * 16
        p, f, b = qv.plan_passes(n, ops.tobytes())
        p1, _, b1 = qv.plan_passes(n, ops.tobytes(), fuse=False)
        assert p <= p1 and f <= p
        assert b >= f * full and b - f * full <= b1
        if f == p:
            assert b == p * full


def test_default_tile_kernels_do_not_spill():
    """The fused tile kernels' default complex128 instantiations (16-amplitude
    subcubes, 128 threads, every class set) sit on a register cliff: a spill of
    a few bytes costs 9-17%. The build's ptxas logs must show none
    for k_tile and k_tile_ahead."""
    import glob
    logs = sorted(glob.glob(os.path.join(ROOT, "paper_2508_15545_b200", "build", "tile_double_*.ptxas.log")))
    if not logs:
        pytest.skip("no ptxas logs (the library was not built by the in-tree Makefile)")
    seen = 0
    for path in logs:
        lines = open(path).read().splitlines()
        for i, line in enumerate(lines):
            m = re.search(r"Compiling entry function '_ZN3qvg(6k_tile|12k_tile_ahead)IdLi4ELb0ELi128E", line)
            if not m:
                continue
            props = " ".join(lines[i + 1:i + 4])
            assert "0 bytes spill stores, 0 bytes spill loads" in props, (path, m.group(1), props)
            assert "Used 96 registers" in props or re.search(r"Used (8\d|9[0-5]) registers", props), props
            seen += 1
    assert seen == 2 * len(logs)


def test_planner_rejects_bad_ops(qv):
    with pytest.raises(qv.ValidationError):
        qv.plan_passes(3, qv.parse_circuit("qubits 4\nh 3\n").gates())


# --- the C-ABI boundary --------------------------------------------------------------
def header_functions():
    with open(os.path.join(ROOT, "include", "qvg.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(qvg_\w+)\s*\(", src, re.M)))


def test_capi_exports_every_declared_symbol(qv):
    lib = ctypes.CDLL(qv.LIBQVG)
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    lib.qvg_abi_version.restype = ctypes.c_int
    assert lib.qvg_abi_version() == qv.QVG_ABI_VERSION == 3
    for name in ("qvg_exchange_plan", "qvg_set_step_hook"):
        assert name in names


@pytest.mark.skipif(cuda_present(), reason="checks the no-device error path")
def test_no_device_fails_loudly(qv):
    lib = ctypes.CDLL(qv.LIBQVG)
    lib.qvg_last_error.restype = ctypes.c_char_p
    st = ctypes.c_void_p()
    rc = lib.qvg_create(4, 128, 0, ctypes.byref(st))
    assert rc in (3, 5) and not st.value and lib.qvg_last_error()
    with pytest.raises(qv.IoError):
        qv.StateVector.create(4)


def test_capi_validation_codes(qv):
    lib = ctypes.CDLL(qv.LIBQVG)
    lib.qvg_last_error.restype = ctypes.c_char_p
    out = ctypes.c_uint64()
    g = np.zeros(1, GATE_DTYPE)
    g[0]["target"] = 5
    g[0]["control"] = -1
    rc = lib.qvg_plan_passes(4, 128, 1, 0, 3, g.ctypes.data_as(ctypes.c_void_p), 1, ctypes.byref(out), None, None)
    assert rc == 1 and b"target 5" in lib.qvg_last_error()
    rc = lib.qvg_create(4, 96, 0, ctypes.byref(ctypes.c_void_p()))
    assert rc == 1


def test_jit_sources_compile_without_gpu(qv):
    """The JIT path's generated sources (one per fused pass, csrc/qvg_jit.cu)
    compile with NVRTC for sm_100a on a host without a GPU: config-shaped
    circuits in both precisions (c64 uses 32-amplitude subcubes)."""
    import shutil
    if not (os.path.exists("/usr/local/cuda/lib64/libnvrtc.so.12") or shutil.which("nvcc")):
        pytest.skip("no NVRTC in this image")
    for c in (qv.qft_circuit(14, 1)[0], qv.grid_circuit(3, 4, 4, 1), qv.u3_ladder_circuit(13, 2, 1)):
        for prec in (128, 64):
            passes, compiled, err = qv.jit_check(c.n_qubits, c.gates(), prec)
            assert passes > 0
            assert compiled == passes, err
