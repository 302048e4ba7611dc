"""BASELINE configs at (or near) full size on the GPU (SURVEY §8d "parity per
config"). Where the CPU oracle cannot finish in seconds, size-independent
properties stand in: an analytic QFT, forward-then-inverse round trips,
fused == per-gate bit-identity (fusion reorders only bit-exactly), shard-count
invariance (reference tests/acceptance.cpp:196-242), and norm drift
(reference tests/acceptance.cpp:398-419)."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import ROOT, gate_array

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden")


def inverse_gates(gates):
    """U^dagger of every op, in reverse order."""
    inv = gates[::-1].copy()
    u = inv["u"].view(np.complex128).reshape(-1, 2, 2)
    inv["u"] = np.ascontiguousarray(np.conj(np.swapaxes(u, 1, 2))).view(np.float64).reshape(-1, 8)
    return inv


def run(qv, circuit, fuse=True, precision=128, world=1):
    st = (qv.StateVector.create(circuit.n_qubits, precision, 0) if world == 1
          else qv.StateVector.create_sharded(circuit.n_qubits, precision, 0, 0, world, None))
    m = qv.apply_circuit(st, circuit, fuse=fuse)
    return st, m


@pytest.mark.parametrize("name", ["config0_u3_ladder_n20", "config1_qft_n16", "config2_haar_sweep_n20",
                                  "config3_grid_4x5_c12", "config4_u3_ladder_n18_l4"])
def test_configs_match_reference_fixture(qv, oracle, name):
    """GPU vs the reference engine's own output (tests/golden/ref_configs.json):
    same op bytes, state equal to the oracle bit for bit, norm and top-8 from
    the reference within 1e-15."""
    with open(os.path.join(GOLD, "ref_configs.json")) as f:
        fx = json.load(f)[name]
    out = getattr(qv, fx["builder"])(*fx["args"])
    c = out[0] if isinstance(out, tuple) else out
    ops = gate_array(c)
    assert hashlib.sha256(ops.tobytes()).hexdigest() == fx["ops_sha256"]
    want = oracle.simulate(c.n_qubits, ops)
    assert hashlib.sha256(want.tobytes()).hexdigest() == fx["state_sha256"]  # oracle == reference
    for fuse in (True, False):
        st, _ = run(qv, c, fuse)
        got = st.read_state()
        assert np.array_equal(got, want), (name, fuse)
        assert abs(st.norm() - fx["norm"]) <= 1e-13
        top = st.top_amplitudes(8)
        assert [i for i, _ in top] == fx["top8_index"]
        assert all(abs(v - complex(*w)) <= 1e-15 for (_, v), w in zip(top, fx["top8"]))


def test_config1_qft_n26_analytic(qv):
    """Config 1 at full size (n=26): the QFT of a seeded basis state |b> has
    amplitude 2^(-n/2) exp(2 pi i b y / 2^n) at every y."""
    n = 26
    c, b = qv.qft_circuit(n, 1, h_layer=False)
    st, m = run(qv, c)
    got = st.read_state()
    y = np.arange(1 << n, dtype=np.float64)
    phase = 2.0 * np.pi * np.mod(b * y, 2.0 ** n) / 2.0 ** n
    want = np.exp(1j * phase) * 2.0 ** (-n / 2)
    assert np.abs(got - want).max() <= 1e-12
    assert abs(st.norm() - 1.0) <= 1e-10


def test_config1_full_circuit_n26_fused_equals_pergate(qv):
    c, _ = qv.qft_circuit(26, 1)
    assert len(c) >= 26 + 26 + 325 + 39
    a, ma = run(qv, c, fuse=True)
    s_f = a.read_state()
    del a
    p, mp = run(qv, c, fuse=False)
    assert np.array_equal(s_f, p.read_state())
    assert ma["traversals"] < mp["traversals"]
    assert abs(p.norm() - 1.0) <= 1e-10


@pytest.mark.parametrize("precision,tol", [(128, 1e-12), (64, 1e-5)])
def test_config2_n30_round_trip(qv, precision, tol):
    """Config 2 at n=30: the Haar+CX sweep followed by its inverse returns to
    |0...0> (within the north_star tolerance for the precision)."""
    n = 30
    c = qv.haar_sweep_circuit(n, 2508)
    g = gate_array(c)
    st = qv.StateVector.create(n, precision, 0)
    st.set_option(qv.OPT_FUSE, 0)
    st.apply_gates(g.tobytes())
    st.apply_gates(inverse_gates(g).tobytes())
    head = st.read_state(0, 1 << 16)
    assert abs(head[0] - 1.0) <= tol
    assert np.abs(head[1:]).max() <= tol
    assert abs(st.norm() - 1.0) <= (1e-10 if precision == 128 else 1e-5)


def test_config3_n30_fused_equals_pergate(qv):
    """Config 3 (5x6 grid, 24 cycles, n=30): the fused planner moves ops only
    where the move keeps every bit (CZ sign flips past ops on other qubits),
    so fused and per-gate runs are bit-identical at full size."""
    c = qv.grid_circuit(5, 6, 24, 1)
    a, ma = run(qv, c, fuse=True)
    fused = a.read_state()
    del a
    b, mb = run(qv, c, fuse=False)
    assert ma["traversals"] * 8 < mb["traversals"]
    chunk = 1 << 26
    for off in range(0, 1 << 30, chunk):
        assert np.array_equal(fused[off:off + chunk], b.read_state(off, chunk)), off
    assert abs(b.norm() - 1.0) <= 1e-10


@pytest.mark.parametrize("world", [2, 8])
def test_config4_shard_invariance_n28(qv, world):
    """Config 4's layer circuit on a sharded state (virtual shards on one GPU):
    bit-identical to the unsharded run; exchanges happen in every layer."""
    n = 28
    c = qv.u3_ladder_circuit(n, 4, 4)
    a, _ = run(qv, c)
    want = a.read_state()
    del a
    st, m = run(qv, c, world=world)
    assert m["exchanges"] >= 4
    assert np.array_equal(st.read_state(), want)


def test_config1_n26_bit_exact_vs_oracle(qv, oracle):
    """Config 1 at full size (n=26, H + QFT + SWAPs, 430 ops) against the
    oracle (OpenMP over disjoint pairs, same bits as the reference's loop)."""
    c, _ = qv.qft_circuit(26, 1)
    want = oracle.simulate(26, gate_array(c))
    for fuse in (True, False):
        st, _ = run(qv, c, fuse)
        assert np.array_equal(st.read_state(), want), fuse
        del st


def test_config2_n28_bit_exact_vs_oracle(qv, oracle):
    """The config-2 sweep shape at n=28 (Haar U on every qubit + CX for
    |c-t| in {1,15}) against the oracle, fused and per gate."""
    c = qv.haar_sweep_circuit(28, 2508)
    want = oracle.simulate(28, gate_array(c))
    for fuse in (True, False):
        st, _ = run(qv, c, fuse)
        assert np.array_equal(st.read_state(), want), fuse
        del st


def test_config3_grid_n24_bit_exact_vs_oracle(qv, oracle):
    """Config 3's generator on a 4x6 grid (n=24, 24 cycles of sqrt-X/Y/W and
    CZ patterns, ~830 ops) against the oracle, fused and per gate."""
    c = qv.grid_circuit(4, 6, 24, 1)
    assert c.n_qubits == 24
    want = oracle.simulate(24, gate_array(c))
    for fuse in (True, False):
        st, m = run(qv, c, fuse)
        assert np.array_equal(st.read_state(), want), fuse
        del st


@pytest.mark.parametrize("world", [4, 8])
def test_config4_layers_n24_sharded_bit_exact_vs_oracle(qv, oracle, world):
    """Config 4's layer circuit at n=24 over 4 / 8 virtual shards (batched and
    pairwise exchanges) against the oracle."""
    c = qv.u3_ladder_circuit(24, 6, 4)
    want = oracle.simulate(24, gate_array(c))
    for batch in (1, 4):
        st = qv.StateVector.create_sharded(24, 128, 0, 0, world, None)
        st.set_option(qv.OPT_BATCH_EXCHANGE, batch)
        m = qv.apply_circuit(st, c)
        assert m["exchanges"] > 0
        assert np.array_equal(st.read_state(), want), (world, batch)
        del st
