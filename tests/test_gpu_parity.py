"""CUDA path vs the oracle (the reference's algorithm, oracle/qv_oracle.c) on
seeded inputs. complex128 must be BIT-IDENTICAL (np.array_equal; the
reference's own engines compare with `== 0.0`, reference
tests/test_kernel.cpp:223-251); complex64 within 1e-5 of the complex128
oracle (north_star tolerance). Every call goes through the C-ABI (libqvg.so)
via the host module."""
import numpy as np
import pytest

from conftest import gate_array

pytestmark = pytest.mark.gpu


def run_gpu(qv, circuit, precision=128, fuse=True, tile_qubits=0, init=None, world=1):
    if world == 1:
        st = qv.StateVector.create(circuit.n_qubits, precision, 0)
    else:
        st = qv.StateVector.create_sharded(circuit.n_qubits, precision, 0, 0, world, None)
    if init is not None:
        st.load_state(init)
    qv.apply_circuit(st, circuit, strategy="gpu", fuse=fuse, tile_qubits=tile_qubits)
    return st, st.read_state()


# --- reference verify-style trials (reference engine.cpp:253-340) -----------------
@pytest.mark.parametrize("fuse", [True, False])
def test_random_circuits_bit_exact(qv, oracle, fuse):
    rng = np.random.default_rng(1)
    for trial in range(60):
        n = int(rng.integers(1, 13))
        depth = int(rng.integers(1, 60))
        c = qv.random_circuit(n, depth, 1000 + trial)
        want = oracle.simulate(n, gate_array(c))
        _, got = run_gpu(qv, c, fuse=fuse)
        assert np.array_equal(got, want), (trial, n, depth, np.abs(got - want).max())


# --- every op flavour on every qubit (reference test_kernel.cpp:223-251) ------------
@pytest.mark.parametrize("n", [6, 9, 14])
def test_each_gate_kind_every_qubit(qv, oracle, n):
    start_c = qv.random_circuit(n, 40, 21)
    start = oracle.simulate(n, gate_array(start_c))
    lines = [f"qubits {n}"]
    for k in range(n):
        lines += [f"h {k}", f"rz {k} 0.7", f"cx {(k + 3) % n} {k}", f"cz {(k + 1) % n} {k}",
                  f"cp {(k + 2) % n} {k} 0.3", f"t {k}", f"x {k}", f"cx {(k + n - 1) % n} {k}"]
    for line in lines[1:]:
        c = qv.parse_circuit(f"qubits {n}\n{line}\n")
        want = oracle.apply(n, start.copy(), gate_array(c))
        for fuse in (False,):
            _, got = run_gpu(qv, c, fuse=fuse, init=start)
            assert np.array_equal(got, want), (line, np.abs(got - want).max())
    # the whole list fused
    c = qv.parse_circuit("\n".join(lines) + "\n")
    want = oracle.apply(n, start.copy(), gate_array(c))
    for tq in (0, 5, 7):
        _, got = run_gpu(qv, c, fuse=True, tile_qubits=tq, init=start)
        assert np.array_equal(got, want), (tq, np.abs(got - want).max())


def test_x_permutation_pattern(qv):
    # reference test_kernel.cpp:125-140: X on qubit 1 swaps at stride 2.
    st = qv.StateVector.create(3, 128, 0)
    st.load_state(np.arange(1, 9, dtype=np.complex128))
    qv.apply_circuit(st, qv.parse_circuit("qubits 3\nx 1\n"))
    assert np.array_equal(st.read_state().real, [3, 4, 1, 2, 7, 8, 5, 6])


def test_control_is_global_index(qv):
    # reference test_kernel.cpp:142-166: control evaluated on the global index.
    st = qv.StateVector.create(4, 128, 0)
    st.load_state(np.arange(16, dtype=np.complex128))
    qv.apply_circuit(st, qv.parse_circuit("qubits 4\ncx 3 0\n"), fuse=False)
    got = st.read_state().real
    want = np.arange(16.0)
    want[8:] = [9, 8, 11, 10, 13, 12, 15, 14]
    assert np.array_equal(got, want)


# --- BASELINE config 0 (n=20, U3 layers + CX ladder, 780 ops) ------------------------
@pytest.mark.parametrize("fuse", [True, False])
def test_config0_bit_exact(qv, oracle, fuse):
    c = qv.u3_ladder_circuit(20, 20, 1)
    assert len(c) == 780
    want = oracle.simulate(20, gate_array(c))
    st, got = run_gpu(qv, c, fuse=fuse)
    assert np.array_equal(got, want)
    assert np.array_equal(st.probabilities(), oracle.probabilities(want))
    assert abs(st.norm() - oracle.norm(want)) <= 1e-12


def test_complex64_within_1e5(qv, oracle):
    for n, c in [(20, qv.u3_ladder_circuit(20, 20, 1)), (16, qv.haar_sweep_circuit(16, 3)),
                 (12, qv.random_circuit(12, 200, 5))]:
        want = oracle.simulate(n, gate_array(c))
        for fuse in (True, False):
            _, got = run_gpu(qv, c, precision=64, fuse=fuse)
            assert np.abs(got - want).max() <= 1e-5, (n, fuse)


# --- sharded path on one device (virtual shards) must be bit-identical ----------------
@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_shards_bit_identical(qv, oracle, world):
    for c in [qv.u3_ladder_circuit(14, 6, 3), qv.random_circuit(12, 300, 9), qv.haar_sweep_circuit(16, 2)]:
        n = c.n_qubits
        want = oracle.simulate(n, gate_array(c))
        for fuse in (True, False):
            st, got = run_gpu(qv, c, fuse=fuse, world=world)
            assert np.array_equal(got, want), (world, n, fuse)
            assert st.stats()["exchanges"] > 0 or world == 1


@pytest.mark.parametrize("world", [2, 4, 8])
def test_exchange_transports_bit_identical(qv, oracle, world):
    """QVG_OPT_EXCHANGE 0 (copy transport: libqvg's chunk plan, D2D copies), 1 (k_xchg, split in two rank-role
    launches like the peer transport) and 2 (k_xchg fused with the gate that
    triggered the exchange, incl. local and global controls), with pairwise
    exchanges only (QVG_OPT_BATCH_EXCHANGE 1) or batched ones (k_mxchg, up to
    3 global qubits at once): all bit-exact with the oracle."""
    circuits = [qv.random_circuit(12, 400, 17), qv.haar_sweep_circuit(14, 5), qv.u3_ladder_circuit(13, 5, 8)]
    for c in circuits:
        n = c.n_qubits
        want = oracle.simulate(n, gate_array(c))
        for batch in (1, 4):
            for mode in (0, 1, 2):
                for fuse in (True, False):
                    st = qv.StateVector.create_sharded(n, 128, 0, 0, world, None)
                    st.set_option(qv.OPT_EXCHANGE, mode)
                    st.set_option(qv.OPT_BATCH_EXCHANGE, batch)
                    qv.apply_circuit(st, c, strategy="gpu", fuse=fuse)
                    s = st.stats()
                    assert np.array_equal(st.read_state(), want), (world, n, batch, mode, fuse)
                    assert s["exchanges"] > 0
                    if batch == 1:
                        assert (s["fused_exchanges"] > 0) == (mode == 2), (mode, s)


@pytest.mark.parametrize("world", [2, 8])
def test_copy_transport_chunk_plan_on_device(qv, oracle, world):
    """Exchange mode 0 on virtual shards runs the NCCL copy transport's chunk
    plan (qvg_exchange_plan) with one D2D copy per chunk and side; chunks of
    48 B / 4 KiB split every run, the default 256 MiB keeps them whole. Both
    pairwise and batched exchanges stay bit-exact with the oracle."""
    c = qv.u3_ladder_circuit(13, 4, 8)
    want = oracle.simulate(13, gate_array(c))
    for chunk in (48, 4096, 0):
        for batch in (1, 4):
            st = qv.StateVector.create_sharded(13, 128, 0, 0, world, None)
            st.set_option(qv.OPT_EXCHANGE, 0)
            st.set_option(qv.OPT_XCHG_CHUNK, chunk)
            st.set_option(qv.OPT_BATCH_EXCHANGE, batch)
            qv.apply_circuit(st, c)
            assert st.stats()["exchanges"] > 0
            assert np.array_equal(st.read_state(), want), (world, chunk, batch)
    with pytest.raises(qv.ValidationError):
        st.set_option(qv.OPT_XCHG_CHUNK, 40)


def test_sharded_timing_splits_passes_and_exchanges(qv):
    """QVG_OPT_TIMING on a sharded state times every segment with CUDA events:
    local pass batches -> kernel_ms, exchanges -> exchange_ms."""
    c = qv.u3_ladder_circuit(20, 3, 2)
    st = qv.StateVector.create_sharded(20, 128, 0, 0, 4, None)
    st.set_option(qv.OPT_TIMING, 1)
    qv.apply_circuit(st, c)
    s = st.stats()
    assert s["exchanges"] > 0 and s["kernel_ms"] > 0 and s["exchange_ms"] > 0
    u = qv.StateVector.create(20, 128, 0)
    u.set_option(qv.OPT_TIMING, 1)
    qv.apply_circuit(u, c)
    assert u.stats()["kernel_ms"] > 0 and u.stats()["exchange_ms"] == 0


def _hook_lib(qv):
    import ctypes

    lib = ctypes.CDLL(qv.LIBQVG)
    fn_t = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32,
                            ctypes.c_uint32)
    lib.qvg_set_step_hook.argtypes = [ctypes.c_void_p, fn_t, ctypes.c_void_p]
    return lib, fn_t


def test_step_hooks_barrier_stagger_and_fault(qv, oracle):
    """The reference's ExecHooks tests (test_parallel.cpp:178-235) on the
    sharded executor: (1) every rank's segment s ends before any rank's
    segment s+1 starts, with rank 0 staggered by a sleep, and the result stays
    bit-exact; (2) an injected fault on rank 1 at segment 2 fails the apply
    with IoError and no later segment starts."""
    import time

    lib, fn_t = _hook_lib(qv)
    c = qv.u3_ladder_circuit(12, 3, 4)
    want = oracle.simulate(12, gate_array(c))
    st = qv.StateVector.create_sharded(12, 128, 0, 0, 4, None)
    start, end = {}, {}

    def hook(user, rank, seg, typ, phase):  # noqa: ARG001
        now = time.perf_counter()
        if phase == 1 and rank == 0:
            time.sleep(0.003)
            now = time.perf_counter()
        book = start if phase == 0 else end
        if phase == 0:
            book[seg] = min(book.get(seg, now), now)
        else:
            book[seg] = max(book.get(seg, now), now)
        return 0

    cb = fn_t(hook)
    assert lib.qvg_set_step_hook(st.handle(), cb, None) == 0
    qv.apply_circuit(st, c)
    s0, e0 = dict(start), dict(end)  # this apply's segments (the readout runs its own)
    assert len(s0) == len(e0) >= 3 and st.stats()["exchanges"] > 0
    for k in range(len(s0) - 1):
        assert e0[k] <= s0[k + 1]
    assert np.array_equal(st.read_state(), want)

    seen = []

    def faulty(user, rank, seg, typ, phase):
        seen.append((seg, rank, phase))
        return 1 if (rank == 1 and seg == 2 and phase == 0) else 0

    st2 = qv.StateVector.create_sharded(12, 128, 0, 0, 4, None)
    cb2 = fn_t(faulty)
    lib.qvg_set_step_hook(st2.handle(), cb2, None)
    with pytest.raises(qv.IoError, match="injected fault"):
        qv.apply_circuit(st2, c)
    assert max(s for s, _, _ in seen) == 2
    assert not any(s == 2 and p == 1 for s, _, p in seen)
    assert lib.qvg_set_step_hook(st2.handle(), fn_t(), None) == 0  # a NULL hook: removed, runs again
    st2.init_basis(0)
    qv.apply_circuit(st2, c)
    assert np.array_equal(st2.read_state(), want)


def test_exchange_fused_complex64(qv, oracle):
    c = qv.haar_sweep_circuit(14, 6)
    want = oracle.simulate(14, gate_array(c))
    for mode, batch in ((0, 1), (2, 1), (1, 4)):
        st = qv.StateVector.create_sharded(14, 64, 0, 0, 4, None)
        st.set_option(qv.OPT_EXCHANGE, mode)
        st.set_option(qv.OPT_BATCH_EXCHANGE, batch)
        qv.apply_circuit(st, c, strategy="gpu")
        assert np.abs(st.read_state() - want).max() <= 1e-5
    with pytest.raises(qv.ValidationError):
        st.set_option(qv.OPT_EXCHANGE, 3)


# --- readout ---------------------------------------------------------------------------
def test_readout(qv, oracle):
    c = qv.random_circuit(10, 80, 3)
    want = oracle.simulate(10, gate_array(c))
    st, _ = run_gpu(qv, c)
    p = oracle.probabilities(want)
    assert np.array_equal(st.probabilities(), p)
    assert np.array_equal(st.probabilities(offset=100, count=50), p[100:150])
    top = st.top_amplitudes(5)
    order = sorted(range(len(p)), key=lambda i: (-p[i], i))[:5]
    assert [i for i, _ in top] == order
    assert abs(st.norm() - oracle.norm(want)) <= 1e-13
    assert st.amplitude(7) == want[7]


def test_ghz_bell(qv):
    st = qv.StateVector.create(3, 128, 0)
    m = qv.apply_circuit(st, qv.parse_circuit("qubits 3\nh 0\ncx 0 1\ncx 1 2\n"), fuse=False)
    assert m["gates_applied"] == 3 and m["traversals"] == 3 and m["strategy"] == "gpu"
    s = st.read_state()
    r = 1 / np.sqrt(2)
    assert abs(s[0] - r) < 1e-15 and abs(s[7] - r) < 1e-15
    assert sorted(i for i, _ in st.top_amplitudes(2)) == [0, 7]


def test_errors_are_typed(qv):
    st = qv.StateVector.create(3, 128, 0)
    with pytest.raises(qv.ValidationError):
        st.apply_gates(qv.parse_circuit("qubits 5\nh 4\n").gates())
    with pytest.raises(qv.ValidationError):
        qv.apply_circuit(st, qv.parse_circuit("qubits 4\nh 0\n"))
    with pytest.raises(qv.ValidationError):
        qv.apply_circuit(st, qv.parse_circuit("qubits 3\nh 0\n"), strategy="paired-cached")
    with pytest.raises(qv.QvsimError):
        qv.StateVector.create(3, 96, 0)


def test_fma_mode_within_tolerance(qv, oracle):
    """QVG_OPT_FMA (opt-in DFMA tile arithmetic) is not bit-exact but stays
    within the north_star 1e-12 of the reference algorithm."""
    for c in [qv.u3_ladder_circuit(20, 20, 1), qv.grid_circuit(4, 5, 12, 3), qv.random_circuit(12, 300, 7)]:
        n = c.n_qubits
        want = oracle.simulate(n, gate_array(c))
        st = qv.StateVector.create(n, 128, 0)
        st.set_option(qv.OPT_FMA, 1)
        qv.apply_circuit(st, c)
        got = st.read_state()
        assert np.abs(got - want).max() <= 1e-12


@pytest.mark.parametrize("sub,pf,k,stage", [(3, 0, 11, 3), (4, 0, 11, 3), (3, 1, 11, 3), (3, 1, 12, 2), (3, 1, 9, 3),
                                             (3, 1, 11, 1), (4, 0, 11, 0), (4, 0, 12, 1), (4, 0, 8, 2), (3, 1, 10, 0)])
def test_tile_subcube_variants_bit_exact(qv, oracle, sub, pf, k, stage):
    """Register subcube 2^3 / 2^4, cp.async next-tile prefetch, tile sizes,
    first/last-group staging through shared memory."""
    for c in [qv.u3_ladder_circuit(16, 6, 2), qv.grid_circuit(3, 5, 10, 4), qv.qft_circuit(14, 3)[0],
              qv.random_circuit(15, 500, 12)]:
        n = c.n_qubits
        want = oracle.simulate(n, gate_array(c))
        st = qv.StateVector.create(n, 128, 0)
        st.set_option(qv.OPT_SUB_BITS, sub)
        st.set_option(qv.OPT_PREFETCH, pf)
        st.set_option(qv.OPT_STAGE, stage)
        st.set_option(qv.OPT_TILE_QUBITS, k)
        m = qv.apply_circuit(st, c, tile_qubits=k)
        assert m["fused_passes"] > 0
        assert np.array_equal(st.read_state(), want)


def test_timing_and_async_copies(qv):
    """QVG_OPT_TIMING fills kernel_ms; load_async/read_async round-trip."""
    n = 16
    st = qv.StateVector.create(n, 128, 0)
    st.set_option(qv.OPT_TIMING, 1)
    qv.apply_circuit(st, qv.make_benchmark_circuit(n))
    assert st.stats()["kernel_ms"] > 0.0
    host = np.random.default_rng(0).standard_normal(2 << n).view(np.complex128)
    st.load_async(host)
    out = np.empty_like(host)
    st.read_async(out)
    st.sync()
    assert np.array_equal(out, host)


def test_verify_equivalence(qv):
    """The reference's verify_equivalence draws (reference engine.cpp:253-340)
    through every device configuration: each must equal the one-pass-per-gate
    run bit for bit (max deviation exactly 0)."""
    r = qv.verify_equivalence(max_qubits=12, trials=60, max_depth=40, seed=3)
    assert r["passed"] and r["failures"] == 0 and r["failure_details"] == []
    assert r["trials"] == 60 and r["comparisons"] >= 150
    assert r["max_deviation"] == 0.0
    with pytest.raises(qv.ValidationError):
        qv.verify_equivalence(max_qubits=30)


# --- property test: every option combination stays bit-exact -------------------------
from hypothesis import HealthCheck, given, settings, strategies as hs  # noqa: E402


@settings(max_examples=80, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(n=hs.integers(2, 14), depth=hs.integers(1, 150), seed=hs.integers(0, 2**32 - 1),
       fuse=hs.booleans(), tile=hs.integers(5, 12), sub=hs.sampled_from([3, 4]), stage=hs.integers(0, 3),
       g=hs.integers(0, 2), exchange=hs.integers(0, 2), batch=hs.sampled_from([1, 4]), graph=hs.booleans(),
       grid=hs.integers(-1, 1), perm=hs.booleans(), pipe=hs.sampled_from([-1, 0, 2, 4, 5, 5, 6]),
       jit=hs.sampled_from([0, 0, 0, 3]))
def test_random_options_bit_exact(qv, oracle, n, depth, seed, fuse, tile, sub, stage, g, exchange, batch, graph,
                                  grid, perm, pipe, jit):
    if n < 2 * g + 2:
        g = 0
    c = qv.random_circuit(n, depth, seed)
    want = oracle.simulate(n, gate_array(c))
    st = (qv.StateVector.create(n, 128, 0) if g == 0
          else qv.StateVector.create_sharded(n, 128, 0, 0, 1 << g, None))
    for key, val in ((qv.OPT_SUB_BITS, sub), (qv.OPT_STAGE, stage), (qv.OPT_EXCHANGE, exchange),
                     (qv.OPT_BATCH_EXCHANGE, batch), (qv.OPT_GRAPH, int(graph)), (qv.OPT_TILE_GRID, grid),
                     (qv.OPT_PERM, int(perm)), (qv.OPT_PIPE, pipe), (qv.OPT_JIT, jit)):
        st.set_option(key, val)
    for _ in range(2 if graph else 1):  # a graph replays on the second run
        st.init_basis(0)
        qv.apply_circuit(st, c, fuse=fuse, tile_qubits=tile)
        assert np.array_equal(st.read_state(), want), (n, depth, seed, fuse, tile, sub, stage, g)


# --- direct parity with the unmodified reference engine (oracle/_ref) ----------------
def test_bit_exact_vs_reference_engine_live(qv):
    """The reference's own engine (compiled from its sources into oracle/_ref,
    strategy paired-cached-parallel) and the GPU path on the same seeded
    circuits at n = 10..18: identical amplitudes, bit for bit."""
    from oracle.oracle import RefEngine

    if not RefEngine.available():
        pytest.skip("oracle/_ref not built")
    eng = RefEngine()
    rng = np.random.default_rng(11)
    for trial in range(16):
        n = int(rng.integers(10, 19))
        c = qv.random_circuit(n, int(rng.integers(50, 400)), 500 + trial)
        with eng.store(n, block_amps=1 << min(n - 2, 14)) as ref:
            ref.apply(gate_array(c), "paired-cached-parallel", 4, 4 * 4 * (16 << min(n - 2, 14)))
            want = ref.read()
        for fuse in (True, False):
            st = qv.StateVector.create(n, 128, 0)
            qv.apply_circuit(st, c, fuse=fuse)
            assert np.array_equal(st.read_state(), want), (trial, n, fuse)


def test_reorder_modes(qv, oracle):
    """QVG_OPT_REORDER. 2 (default): only bit-exact moves (an X/CX permutation
    or a Z/CZ sign flip on either side), results bit-identical to the oracle.
    1 (opt-in): any move across disjoint qubits, amplitudes within 1e-12 of the
    oracle (the reference's verify tolerance, reference engine.hpp:93) and
    fidelity 1 - 1e-12. Passes: 1 <= 2 <= 0 (circuit order)."""
    cases = [qv.grid_circuit(3, 5, 24, 2), qv.u3_ladder_circuit(15, 8, 3), qv.random_circuit(14, 600, 8),
             qv.qft_circuit(15, 2)[0], qv.haar_sweep_circuit(16, 9)]
    for c in cases:
        n = c.n_qubits
        want = oracle.simulate(n, gate_array(c))
        passes = {}
        for reorder in (0, 1, 2):
            st = qv.StateVector.create(n, 128, 0)
            st.set_option(qv.OPT_REORDER, reorder)
            m = qv.apply_circuit(st, c)
            passes[reorder] = m["traversals"]
            got = st.read_state()
            if reorder == 1:
                assert np.abs(got - want).max() <= 1e-12, n
                assert abs(np.vdot(want, got)) ** 2 >= 1 - 1e-12
            else:
                assert np.array_equal(got, want), (n, reorder, np.abs(got - want).max())
        assert passes[1] <= passes[2] <= passes[0], (n, passes)


# --- structured-matrix op bodies in fused tiles (QVG_OPT_CLASSES, qvg_tile.cuh) ---
@pytest.mark.parametrize("n", [7, 12, 16])
def test_structured_classes_bit_exact(qv, oracle, n):
    """Real (H, ry), X (x, the CX target), entries +-1/2 (sx, sy and adjoint-like
    sign patterns as `u`/`cu`) and Z/CZ take the reduced-FP64 bodies; results
    are bit-identical to the oracle and to the general bodies, for every
    register slot / control slot combination the planner produces."""
    start = oracle.simulate(n, gate_array(qv.random_circuit(n, 30, 5)))
    half = ["0.5 0.5 0.5 -0.5 0.5 -0.5 0.5 0.5", "0.5 -0.5 0.5 0.5 0.5 0.5 0.5 -0.5",
            "0.5 0.5 -0.5 -0.5 0.5 0.5 0.5 0.5", "0.5 -0.5 0.5 -0.5 -0.5 0.5 0.5 -0.5"]
    lines = [f"qubits {n}"]
    for k in range(n):
        c = (k + 1 + k % 3) % n
        lines += [f"sx {k}", f"h {k}", f"cx {c} {k}", f"sy {k}", f"cz {c} {k}", f"z {k}",
                  f"u {k} {half[k % 4]}", f"cu {c} {k} {half[(k + 1) % 4]}", f"ry {k} 0.4", f"x {k}",
                  f"sw {k}", f"cx {k} {(k + 5) % n}"]
    circ = qv.parse_circuit("\n".join(lines) + "\n")
    want = oracle.apply(n, start.copy(), gate_array(circ))
    for classes in (1, 0):
        for tq, sub in ((0, 4), (7, 3), (5, 3)):
            st = qv.StateVector.create(n, 128, 0)
            st.load_state(start)
            st.set_option(qv.OPT_CLASSES, classes)
            st.set_option(qv.OPT_SUB_BITS, sub)
            qv.apply_circuit(st, circ, strategy="gpu", fuse=True, tile_qubits=tq)
            got = st.read_state()
            assert np.array_equal(got, want), (classes, tq, sub, np.abs(got - want).max())
    st = qv.StateVector.create(n, 64, 0)
    st.load_state(start.astype(np.complex64))
    qv.apply_circuit(st, circ, strategy="gpu", fuse=True)
    assert np.abs(st.read_state() - want).max() <= 1e-5


@pytest.mark.parametrize("n", [8, 13])
def test_grid_gate_set_bit_exact(qv, oracle, n):
    """Passes of sqrt(X)/sqrt(Y)/sqrt(W) + CZ only (config 3's gate set) take the
    {general, +-1/2, sqrt(W)} body set; bit-identical to the oracle, with
    every register-slot and control-slot combination."""
    start = oracle.simulate(n, gate_array(qv.random_circuit(n, 20, 8)))
    rng = np.random.default_rng(n)
    lines = [f"qubits {n}"]
    for _ in range(12):
        for k in range(n):
            lines.append(f"{['sx', 'sy', 'sw'][int(rng.integers(3))]} {k}")
        for k in range(n):
            c = int(rng.integers(n))
            if c != k:
                lines.append(f"cz {c} {k}")
                lines.append(f"cu {c} {k} 0.5 0.5 0 -0.7071067811865476 0.7071067811865476 0 0.5 0.5")
    circ = qv.parse_circuit("\n".join(lines) + "\n")
    want = oracle.apply(n, start.copy(), gate_array(circ))
    for tq, sub in ((0, 4), (6, 3)):
        st = qv.StateVector.create(n, 128, 0)
        st.load_state(start)
        st.set_option(qv.OPT_SUB_BITS, sub)
        qv.apply_circuit(st, circ, strategy="gpu", fuse=True, tile_qubits=tq)
        got = st.read_state()
        assert np.array_equal(got, want), (tq, sub, np.abs(got - want).max())


def test_subcube_option_bounds(qv, oracle):
    """QVG_OPT_SUB_BITS: complex128 takes 3..4, complex64 3..5 (its default is
    5: 32 register amplitudes); a complex64 run at each size stays within
    1e-5 of the oracle."""
    st = qv.StateVector.create(10, 128, 0)
    with pytest.raises(qv.ValidationError):
        st.set_option(qv.OPT_SUB_BITS, 5)
    c = qv.random_circuit(13, 200, 4)
    want = oracle.simulate(13, gate_array(c))
    for sub in (3, 4, 5):
        st = qv.StateVector.create(13, 64, 0)
        st.set_option(qv.OPT_SUB_BITS, sub)
        qv.apply_circuit(st, c)
        assert np.abs(st.read_state() - want).max() <= 1e-5, sub
    with pytest.raises(qv.ValidationError):
        qv.StateVector.create(10, 64, 0).set_option(qv.OPT_SUB_BITS, 6)


# --- JIT-specialised fused passes (QVG_OPT_JIT, csrc/qvg_jit.hpp) -------------------
@pytest.mark.parametrize("prec", [128, 64])
def test_jit_passes_bit_exact(qv, oracle, prec):
    """Every fused pass compiled before launch (mode 3) as a kernel specialised
    to its op list: complex128 bit-identical to the oracle, complex64 within
    1e-5 and bit-identical to k_tile; the passes did run as JIT kernels."""
    rng = np.random.default_rng(5)
    for trial in range(12):
        n = int(rng.integers(6, 15))
        c = qv.random_circuit(n, int(rng.integers(20, 120)), 7000 + trial)
        want = oracle.simulate(n, gate_array(c))
        st = qv.StateVector.create(n, prec, 0)
        st.set_option(qv.OPT_JIT, 3)
        m = qv.apply_circuit(st, c, fuse=True)
        got = st.read_state()
        if m["fused_passes"]:
            assert st.stats()["jit_passes"] == m["fused_passes"], (trial, st.stats())
        if prec == 128:
            assert np.array_equal(got, want), (trial, n, np.abs(got - want).max())
        else:
            assert np.abs(got.astype(np.complex128) - want).max() <= 1e-5
            ref = qv.StateVector.create(n, prec, 0)
            ref.set_option(qv.OPT_JIT, 0)
            qv.apply_circuit(ref, c, fuse=True)
            assert st.max_deviation(ref) <= 1e-6


def test_jit_config_circuits_and_graphs(qv, oracle):
    """The BASELINE circuit shapes (QFT, grid, U3 ladder, Haar sweep) at n = 16
    through JIT kernels on every pass (mode 3), applied once and then replayed
    as captured CUDA graphs that hold the JIT kernels: bit-identical to the
    oracle on every apply."""
    n = 16
    circs = [qv.qft_circuit(n, 3)[0], qv.grid_circuit(4, 4, 8, 2), qv.u3_ladder_circuit(n, 3, 4),
             qv.haar_sweep_circuit(n, 9)]
    for ci, c in enumerate(circs):
        want = oracle.simulate(n, gate_array(c))
        st = qv.StateVector.create(n, 128, 0)
        st.set_option(qv.OPT_JIT, 3)
        qv.apply_circuit(st, c)
        assert np.array_equal(st.read_state(), want)
        assert st.stats()["jit_passes"] > 0
        st2 = qv.StateVector.create(n, 128, 0)  # graphs auto (captured from the 2nd apply), JIT on every pass
        st2.set_option(qv.OPT_JIT, 3)
        g = c.gates()
        for rep in range(4):
            st2.init_basis(0)
            st2.apply_gates(g)
            assert np.array_equal(st2.read_state(), want), rep
        s2 = st2.stats()
        assert s2["graph_replays"] >= 2 and s2["jit_passes"] > 0, s2


# --- permutation / sign-flip passes (QVG_OPT_PERM, csrc/qvg_tile_perm.cuh) --------
def _perm_circuit(qv, n, seed, mixed):
    rng = np.random.default_rng(seed)
    lines = [f"qubits {n}"] + [f"h {q}" for q in range(0, n, 2)] + [f"ry {q} 0.4" for q in range(1, n, 3)]
    for _ in range(60):
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        kind = int(rng.integers(6 if mixed else 5))
        lines.append([f"x {a}", f"cx {a} {b}", f"z {a}", f"cz {a} {b}", f"swap {a} {b}", f"h {a}"][kind])
    return qv.parse_circuit("\n".join(lines) + "\n")


@pytest.mark.parametrize("prec", [128, 64])
@pytest.mark.parametrize("n", [6, 11, 14, 17])
def test_perm_passes_bit_exact(qv, oracle, prec, n):
    """Runs of X / CX / Z / CZ / SWAP (controls in and outside the tile, sign
    flips on every qubit) through k_tile_perm: in circuit order (QVG_OPT_REORDER
    0) the same BYTES as k_tile (signs of zeros included; the start state has
    exact zeros); with the default reordering (a sign flip and a move may swap,
    which can change the sign of an exact zero only) the same values; and, for
    complex128, the oracle's values."""
    for seed, mixed in ((1, False), (2, True), (3, False)):
        c = _perm_circuit(qv, n, 100 * n + seed, mixed)
        got = {}
        for perm, reorder in ((1, 0), (0, 0), (1, 2), (0, 2)):
            st = qv.StateVector.create(n, prec, 0)
            st.set_option(qv.OPT_PERM, perm)
            st.set_option(qv.OPT_JIT, 0)
            st.set_option(qv.OPT_REORDER, reorder)
            m = qv.apply_circuit(st, c)
            got[perm, reorder] = st.read_state()
        bits = np.uint64 if prec == 128 else np.uint32
        assert np.array_equal(got[1, 0].view(bits), got[0, 0].view(bits)), (seed, mixed)
        assert np.array_equal(got[1, 2], got[0, 2]) and np.array_equal(got[1, 2], got[1, 0]), (seed, mixed)
        got = {1: got[1, 2], 0: got[0, 2]}
        if prec == 128:
            want = oracle.simulate(n, gate_array(c))
            assert np.array_equal(got[1], want)
        else:
            assert np.abs(got[1].astype(np.complex128) - oracle.simulate(n, gate_array(c))).max() <= 1e-5
