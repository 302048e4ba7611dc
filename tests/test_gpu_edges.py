"""Edge cases on the device path: the smallest and empty inputs, range and
capacity errors, basis states, precision mixes, repeated apply calls (plan
buffers reused), and odd tile options (reference tests: test_store.cpp size
checks, test_kernel.cpp:120-123 out-of-range targets, test_parallel.cpp
worker-count edges)."""
import numpy as np
import pytest

from conftest import gate_array

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_tiny_states_every_kernel(qv, oracle, n):
    c = qv.random_circuit(n, 80, 100 + n)
    want = oracle.simulate(n, gate_array(c))
    for fuse in (True, False):
        for prec in (128, 64):
            st = qv.StateVector.create(n, prec, 0)
            qv.apply_circuit(st, c, fuse=fuse)
            got = st.read_state()
            if prec == 128:
                assert np.array_equal(got, want), (n, fuse)
            else:
                assert np.abs(got - want).max() <= 1e-5


def test_empty_circuit_and_identity_ops(qv):
    st = qv.StateVector.create(6, 128, 0)
    m = qv.apply_circuit(st, qv.parse_circuit("qubits 6\n"))
    assert m["gates_applied"] == 0 and m["traversals"] == 0
    m = qv.apply_circuit(st, qv.parse_circuit("qubits 6\ncp 1 2 0\nrz 3 0\n"), fuse=False)
    # cp(0) is the identity (no pass); rz(0) = diag(1,1) as well
    assert m["traversals"] == 0
    s = st.read_state()
    assert s[0] == 1 and not s[1:].any()


def test_basis_init_and_ranges(qv):
    st = qv.StateVector.create(8, 128, 0)
    st.init_basis(200)
    s = st.read_state()
    assert s[200] == 1 and np.count_nonzero(s) == 1
    assert st.amplitude(200) == 1
    with pytest.raises(qv.ValidationError):
        st.init_basis(256)
    with pytest.raises(qv.ValidationError):
        st.read_state(250, 10)
    with pytest.raises(qv.ValidationError):
        st.load_state(np.zeros(10, np.complex128), 250)
    with pytest.raises(qv.ValidationError):
        st.amplitude(256)
    assert st.read_state(256, 0).size == 0


def test_capacity_error_is_typed(qv):
    # 2^40 complex128 amplitudes = 16 TiB: the device allocation must fail as CapacityError
    with pytest.raises(qv.CapacityError):
        qv.StateVector.create(40, 128, 0)
    with pytest.raises(qv.ValidationError):
        qv.StateVector.create(41, 128, 0)


def test_shard_limits(qv):
    with pytest.raises(qv.ValidationError):
        qv.StateVector.create_sharded(3, 128, 0, 0, 4, None)  # too few qubits for 4 shards
    with pytest.raises(qv.ValidationError):
        qv.StateVector.create_sharded(10, 128, 0, 0, 3, None)  # not a power of two
    st = qv.StateVector.create_sharded(4, 128, 0, 0, 4, None)  # L = 2, the minimum
    c = qv.random_circuit(4, 60, 9)
    st2 = qv.StateVector.create(4, 128, 0)
    qv.apply_circuit(st, c)
    qv.apply_circuit(st2, c)
    assert np.array_equal(st.read_state(), st2.read_state())


def test_repeated_apply_reuses_plan_buffers(qv, oracle):
    n = 14
    st = qv.StateVector.create(n, 128, 0)
    want = oracle.basis(n)
    for seed in range(6):
        c = qv.random_circuit(n, 50 + 37 * seed, seed)
        qv.apply_circuit(st, c)
        oracle.apply(n, want, gate_array(c))
    assert np.array_equal(st.read_state(), want)


@pytest.mark.parametrize("opt,val", [("OPT_TILE_QUBITS", 5), ("OPT_TILE_QUBITS", 12), ("OPT_CARRIERS", 0),
                                     ("OPT_CARRIERS", 6), ("OPT_SUB_BITS", 3), ("OPT_LOW_KERNEL", 1),
                                     ("OPT_MIN_RUN", 128), ("OPT_PRED_STORE", 1), ("OPT_PIPE", 2), ("OPT_PIPE", 3),
                                     ("OPT_PIPE", 4), ("OPT_PIPE", 5), ("OPT_PIPE", 6), ("OPT_PIPE", 0),
                                     ("OPT_TILE_GRID", 0), ("OPT_TILE_GRID", 1),
                                     ("OPT_TILE_ORDER", 1), ("OPT_PERM", 1), ("OPT_JIT", 3)])
@pytest.mark.parametrize("prec", [128, 64])
def test_options_keep_bits(qv, oracle, opt, val, prec):
    """Every engine option leaves complex128 bit-identical to the oracle and
    complex64 within 1e-5 (and bit-identical to the default options): the
    pipelines (bulk-copy ring, tensor-map TMA; complex64 passes fall back to
    k_tile there), the load-ahead kernel, tile grid / order, permutation
    passes, JIT passes."""
    n = 15 if opt in ("OPT_PIPE", "OPT_TILE_GRID", "OPT_TILE_ORDER") else 13
    c = qv.random_circuit(n, 400, 77)
    want = oracle.simulate(n, gate_array(c))
    st = qv.StateVector.create(n, prec, 0)
    st.set_option(getattr(qv, opt), val)
    qv.apply_circuit(st, c, tile_qubits=val if opt == "OPT_TILE_QUBITS" else 0)
    got = st.read_state()
    if prec == 128:
        assert np.array_equal(got, want)
    else:
        assert np.abs(got.astype(np.complex128) - want).max() <= 1e-5
        if opt not in ("OPT_TILE_QUBITS", "OPT_SUB_BITS", "OPT_CARRIERS"):  # same tile shapes: same bits
            ref = qv.StateVector.create(n, prec, 0)
            qv.apply_circuit(ref, c)
            assert st.max_deviation(ref) == 0.0


def test_bad_options(qv):
    st = qv.StateVector.create(4, 128, 0)
    for key, val in [(qv.OPT_TILE_QUBITS, 13), (qv.OPT_TILE_QUBITS, 1), (qv.OPT_MIN_RUN, 3),
                     (qv.OPT_SUB_BITS, 5), (999, 1)]:
        with pytest.raises(qv.ValidationError):
            st.set_option(key, val)


def test_nonfinite_matrix_rejected(qv):
    st = qv.StateVector.create(4, 128, 0)
    g = gate_array(qv.parse_circuit("qubits 4\nh 1\n"))
    g[0]["u"][0] = np.nan
    with pytest.raises(qv.ValidationError, match="finite"):
        st.apply_gates(g.tobytes())


@pytest.mark.parametrize("prec", [128, 64])
def test_out_of_core_bit_identical(qv, oracle, prec):
    """qvg_apply_host: state in host memory, 2^w-amplitude HBM windows; the
    result equals the device-resident run bit for bit (c128 also equals the
    oracle), for circuits whose gates hit every qubit."""
    cdt = np.complex128 if prec == 128 else np.complex64
    for c, w in [(qv.u3_ladder_circuit(18, 3, 5), 12), (qv.random_circuit(16, 400, 8), 8),
                 (qv.grid_circuit(4, 5, 6, 2), 14), (qv.qft_circuit(17, 3)[0], 10)]:
        n = c.n_qubits
        dev = qv.StateVector.create(n, prec, 0)
        qv.apply_circuit(dev, c)
        want = dev.read_state().astype(cdt)
        host = np.zeros(1 << n, cdt)
        host[0] = 1
        st = qv.apply_circuit_host(host, c, w)
        assert st["segments"] >= 2 and st["host_bytes"] == st["segments"] * 2 * host.nbytes
        if prec == 128:
            assert np.array_equal(host, want), (n, w)
            assert np.array_equal(host, oracle.simulate(n, gate_array(c)))
        else:  # complex64 contracts to FFMA differently per kernel plan: compare within 1e-6
            assert np.abs(host - want).max() <= 1e-6, (n, w)


def test_states_on_concurrent_host_threads(qv, oracle):
    """One state per host thread (the reference's single-owner rule,
    reference cache.hpp:44-47); several threads may drive their own states at
    once (the GIL is released). Fused passes build their parameter block per
    thread, so concurrent launches do not race."""
    import threading

    circuits = [qv.random_circuit(14, 300, 100 + i) for i in range(4)]
    wants = [oracle.simulate(14, gate_array(c)) for c in circuits]
    got = [None] * len(circuits)
    errors = []

    def work(i):
        try:
            st = qv.StateVector.create(14, 128, 0)
            for _ in range(5):
                st.init_basis(0)
                qv.apply_circuit(st, circuits[i])
            got[i] = st.read_state()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(circuits))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(len(circuits)):
        assert np.array_equal(got[i], wants[i]), i


def test_graph_auto_mode_replays_repeated_circuits(qv, oracle):
    """QVG_OPT_GRAPH 2 (default): a circuit applied once runs eagerly; from its
    second apply on the same state it replays as a captured graph, bit-exact.
    Single-gate calls (the per-gate bench) never capture."""
    n = 16
    c = qv.u3_ladder_circuit(n, 4, 2)
    want = oracle.simulate(n, gate_array(c))
    st = qv.StateVector.create(n, 128, 0)
    for rep in range(3):
        st.init_basis(0)
        qv.apply_circuit(st, c)
        assert np.array_equal(st.read_state(), want), rep
        assert st.stats()["graph_replays"] == rep
    g = gate_array(c)
    for _ in range(3):
        st.apply_gates(g[:1].tobytes())
    assert st.stats()["graph_replays"] == 2
    with pytest.raises(qv.ValidationError):
        st.set_option(qv.OPT_GRAPH, 3)


def test_graph_replay_bit_identical(qv, oracle):
    """QVG_OPT_GRAPH: a repeated op list replays as a captured CUDA graph with
    the same results and pass accounting; a changed option or op list
    captures anew."""
    n = 14
    c = qv.random_circuit(n, 300, 5)
    want = oracle.simulate(n, gate_array(c))
    st = qv.StateVector.create(n, 128, 0)
    st.set_option(qv.OPT_GRAPH, 1)
    passes = []
    for rep in range(3):
        st.init_basis(0)
        st.reset_stats()
        qv.apply_circuit(st, c)
        passes.append(st.stats()["passes"])
        assert np.array_equal(st.read_state(), want), rep
    assert passes[0] == passes[1] == passes[2] > 0
    for fuse in (False, True):  # other plan options -> another graph
        st.init_basis(0)
        qv.apply_circuit(st, c, fuse=fuse)
        assert np.array_equal(st.read_state(), want), fuse
    c2 = qv.random_circuit(n, 50, 6)
    st.init_basis(0)
    qv.apply_circuit(st, c2)
    assert np.array_equal(st.read_state(), oracle.simulate(n, gate_array(c2)))
    st.set_option(qv.OPT_GRAPH, 0)


@pytest.mark.parametrize("prec", [128, 64])
@pytest.mark.parametrize("n", [6, 10, 16])
def test_warp_shuffle_low_kernel_per_gate(qv, oracle, prec, n):
    """k_low (north_star's warp-shuffle pairing for targets < 5, QVG_OPT_LOW_KERNEL)
    with fusion OFF, so every op on qubits 0..4 is its own k_low launch: every
    target 0..4, uncontrolled and with a control below / above the target (the
    inserted and the selected control), general, real and permutation
    matrices. complex128 bit-identical to the oracle, complex64 within 1e-5.
    The CUPTI kernel list (torch.profiler) must show k_low launches, so the
    test cannot pass on k_pairs alone."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    start = oracle.simulate(n, gate_array(qv.random_circuit(n, 30, 5)))
    lines = [f"qubits {n}"]
    for t in range(5):
        lines += [f"u3 {t} 0.3 1.1 -0.4", f"h {t}", f"cx {(t + 1) % n} {t}", f"cx {n - 1} {t}",
                  f"cu {(t + 3) % n} {t} 0.6 0 0 0.8 0 0.8 0.6 0", f"x {t}"]
        if t > 0:
            lines.append(f"cx 0 {t}")
    c = qv.parse_circuit("\n".join(lines) + "\n")
    want = oracle.apply(n, start.copy(), gate_array(c))
    st = qv.StateVector.create(n, prec, 0)
    st.set_option(qv.OPT_LOW_KERNEL, 1)
    st.load_state(start)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        m = qv.apply_circuit(st, c, fuse=False)
        st.sync()
        torch.cuda.synchronize()
    got = st.read_state()
    assert m["traversals"] == len(c)
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    assert sum("k_low" in s for s in names) >= 5 * 5, sorted(set(names))
    if prec == 128:
        assert np.array_equal(got, want), np.abs(got - want).max()
    else:
        assert np.abs(got.astype(np.complex128) - want).max() <= 1e-5


@pytest.mark.parametrize("prec", [128, 64])
@pytest.mark.parametrize("grid", [0, -1])
def test_load_ahead_kernel_several_tiles_per_cta(qv, oracle, prec, grid):
    """k_tile_ahead (QVG_OPT_PIPE 5: the next tile's cp.async load lands in the
    shared tile while the last register group runs) with CTAs that run several
    tiles in a row (n = 22: 2048 tiles on a persistent grid, or the default
    tiles-per-CTA split): complex128 bit-identical to the oracle, complex64
    bit-identical to k_tile; staged first / last groups included (random
    circuits put gates on qubits 0..2)."""
    n = 22
    c = qv.random_circuit(n, 120, 4242)
    st = qv.StateVector.create(n, prec, 0)
    st.set_option(qv.OPT_PIPE, 5)
    st.set_option(qv.OPT_TILE_GRID, grid)
    m = qv.apply_circuit(st, c)
    assert m["traversals"] < len(c)
    if prec == 128:
        want = oracle.simulate(n, gate_array(c))
        assert np.array_equal(st.read_state(), want)
    ref = qv.StateVector.create(n, prec, 0)
    ref.set_option(qv.OPT_PIPE, 0)
    qv.apply_circuit(ref, c)
    assert st.max_deviation(ref) == 0.0


@pytest.mark.parametrize("prec,S", [(128, 16), (64, 8)])
def test_counter_laws_on_device(qv, oracle, prec, S):
    """The reference's single-traversal law as exact equalities on the device
    (proj/tests/test_kernel.cpp:253-277): with
    fusion off every non-identity gate is exactly one HBM pass and one kernel
    launch, and `bytes_moved` is SURVEY §8d's per-gate bytes summed from the
    table; with fusion on the counters equal the planner's (qvg_plan_passes)
    and a fused pass is charged one traversal of the state."""
    from conftest import algorithmic_bytes
    n = 18
    ops, _ = oracle.random_circuit(n, 300, 99)
    gates = ops.tobytes()
    want = [algorithmic_bytes(n, S, op) for op in ops]
    st = qv.StateVector.create(n, prec, 0)
    st.set_option(qv.OPT_GRAPH, 0)
    st.set_option(qv.OPT_FUSE, 0)
    st.apply_gates(gates)
    s = st.stats()
    live = sum(1 for w in want if w)
    assert s["gates_applied"] == len(ops)
    assert s["passes"] == live and s["kernel_launches"] == live and s["fused_passes"] == 0
    assert s["bytes_moved"] == sum(want)
    st.reset_stats()
    st.set_option(qv.OPT_FUSE, 1)
    st.apply_gates(gates)
    s = st.stats()
    p, f, b = qv.plan_passes(n, gates, precision=prec)
    assert (s["passes"], s["fused_passes"], s["bytes_moved"]) == (p, f, b)
    assert s["kernel_launches"] == p and p < live
    assert b >= f * 2 * (1 << n) * S
