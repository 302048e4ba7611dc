"""Device readout: top-k by radix select against
the reference's ordering (|a|^2 descending, ties by ascending index,
reference engine.cpp:511-544), inner product / fidelity and max deviation
against numpy on the same states."""
import numpy as np
import pytest

from conftest import gate_array

pytestmark = pytest.mark.gpu


def ref_topk(state, k):
    p = state.real * state.real + state.imag * state.imag
    order = np.lexsort((np.arange(p.size), -p))[:k]
    return [int(i) for i in order]


@pytest.mark.parametrize("world", [1, 4])
@pytest.mark.parametrize("prec", [128, 64])
def test_topk_matches_reference_order(qv, oracle, world, prec):
    for n, c in [(12, qv.random_circuit(12, 300, 5)), (16, qv.u3_ladder_circuit(16, 3, 2)),
                 (10, qv.parse_circuit("qubits 10\n" + "".join(f"h {q}\n" for q in range(10))))]:
        st = (qv.StateVector.create(n, prec, 0) if world == 1
              else qv.StateVector.create_sharded(n, prec, 0, 0, world, None))
        qv.apply_circuit(st, c)
        state = st.read_state()
        for k in (1, 5, 64, 1 << n, (1 << n) + 3):
            got = st.top_amplitudes(k)
            want = ref_topk(state, k)
            assert [i for i, _ in got] == want, (n, k)
            assert all(v == state[i] for i, v in got)


def test_topk_all_ties_uniform_state(qv):
    # H on every qubit: 2^20 equal probabilities -> the first k indices
    st = qv.StateVector.create(20, 128, 0)
    qv.apply_circuit(st, qv.make_benchmark_circuit(20))
    assert [i for i, _ in st.top_amplitudes(100)] == list(range(100))


def test_topk_basis_and_zero_keys(qv):
    st = qv.StateVector.create(14, 128, 0)
    st.init_basis(9999)
    top = st.top_amplitudes(4)
    assert [i for i, _ in top] == [9999, 0, 1, 2]  # then zeros by index


def test_inner_fidelity_maxdev(qv, oracle):
    n = 14
    a = qv.StateVector.create(n, 128, 0)
    b = qv.StateVector.create(n, 128, 0)
    qv.apply_circuit(a, qv.random_circuit(n, 200, 1))
    qv.apply_circuit(b, qv.random_circuit(n, 200, 2))
    sa, sb = a.read_state(), b.read_state()
    ip = a.inner(b)
    assert abs(ip - np.vdot(sa, sb)) <= 1e-13
    assert abs(a.fidelity(b) - abs(np.vdot(sa, sb)) ** 2) <= 1e-13
    assert a.max_deviation(b) == np.abs(sa - sb).max()
    assert abs(a.fidelity(a) - 1.0) <= 1e-12 and a.max_deviation(a) == 0.0
    with pytest.raises(qv.ValidationError):
        a.inner(qv.StateVector.create(n + 1, 128, 0))


def test_sharded_inner_equals_unsharded(qv):
    n = 14
    c1, c2 = qv.random_circuit(n, 300, 3), qv.random_circuit(n, 300, 4)
    ua, ub = qv.StateVector.create(n, 128, 0), qv.StateVector.create(n, 128, 0)
    sa, sb = qv.StateVector.create_sharded(n, 128, 0, 0, 4, None), qv.StateVector.create_sharded(n, 128, 0, 0, 4, None)
    for s, c in ((ua, c1), (ub, c2), (sa, c1), (sb, c2)):
        qv.apply_circuit(s, c)
    assert abs(sa.inner(sb) - ua.inner(ub)) <= 1e-13
    assert sa.max_deviation(sb) == ua.max_deviation(ub)


@pytest.mark.parametrize("world", [1, 2])
def test_topk_whole_state_with_zero_amplitudes(qv, world):
    """k >= 2^n on states with zero amplitudes: a basis state and a
    GHZ state return every index, the nonzero ones first, then the zeros by
    ascending index."""
    st = (qv.StateVector.create(3, 128, 0) if world == 1
          else qv.StateVector.create_sharded(3, 128, 0, 0, world, None))
    assert [i for i, _ in st.top_amplitudes(8)] == list(range(8))
    ghz = qv.parse_circuit("qubits 4\nh 0\ncx 0 1\ncx 1 2\ncx 2 3\n")
    st = (qv.StateVector.create(4, 128, 0) if world == 1
          else qv.StateVector.create_sharded(4, 128, 0, 0, world, None))
    qv.apply_circuit(st, ghz)
    for k in (16, 20):
        got = st.top_amplitudes(k)
        assert [i for i, _ in got] == [0, 15] + list(range(1, 15)), k
        assert abs(got[0][1] - 2 ** -0.5) <= 1e-15 and got[2][1] == 0
    st.init_basis(5)
    assert [i for i, _ in st.top_amplitudes(16)] == [5] + [i for i in range(16) if i != 5]


@pytest.mark.parametrize("world", [1, 4])
@pytest.mark.parametrize("prec", [128, 64])
def test_device_checksums_match_numpy(qv, world, prec):
    """qvg_checksums equals its numpy restatement on the state read back, for
    sharded (canonicalised first) and unsharded states, both precisions; a
    single flipped bit (the sign of one zero) changes its chunk's words."""
    from conftest import checksums_numpy

    n = 16
    st = (qv.StateVector.create(n, prec, 0) if world == 1
          else qv.StateVector.create_sharded(n, prec, 0, 0, world, None))
    qv.apply_circuit(st, qv.random_circuit(n, 300, 8))
    host = st.read_state()
    if prec == 64:
        host = host.astype(np.complex64)
    for chunk in (4096, 1 << 14, 1 << n):
        assert np.array_equal(st.checksums(chunk), checksums_numpy(host, chunk)), chunk
    z = qv.StateVector.create(n, 128, 0)
    a = z.checksums(4096)
    neg = np.zeros(1 << n, np.complex128)
    neg[0] = 1.0
    neg[5000] = complex(-0.0, 0.0)
    z.load_state(neg)
    b = z.checksums(4096)
    assert (a[1] != b[1]).all() and np.array_equal(np.delete(a, 1, 0), np.delete(b, 1, 0))
    with pytest.raises(qv.ValidationError):
        z.checksums(1000)
