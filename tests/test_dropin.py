"""The reference-side drop-in (VERDICT r1 "missing" #3):
the reference's OWN engine and pybind11 module, rebuilt from copies of its
engine.hpp / engine.cpp with the `Strategy::gpu` branch added
(integration/reference_patch.py, integration/gpu_strategy.cpp, `make -C
oracle dropin`) and linked with libqvg.so. `qvsim.apply_circuit(store, c,
strategy="gpu")` — the reference's binding forwarding the tag to its C++
`apply_circuit(BlockStore&, ...)` — must equal the reference's own
paired-cached engine on the same QVSV file bit for bit."""
import math
import os
import sys

import pytest

from conftest import ROOT

DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin", "python")


@pytest.fixture(scope="module")
def qvsim():
    if not os.path.isdir(os.path.join(DROPIN, "qvsim")):
        pytest.fail("reference drop-in not built: make -C oracle dropin (needs /root/reference once)")
    sys.path.insert(0, DROPIN)
    try:
        import qvsim as mod
    finally:
        sys.path.remove(DROPIN)
    assert mod.__file__.startswith(DROPIN)
    return mod


def cuda_present():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def test_dropin_module_is_the_reference_with_a_gpu_tag(qvsim, tmp_path):
    """CPU: the rebuilt reference module runs its own strategies, knows the
    "gpu" tag, and (without a device) fails it loudly as QvsimError."""
    c = qvsim.parse_circuit("qubits 2\nh 0\ncx 0 1\n")
    st = qvsim.StateStore.create(str(tmp_path / "bell.qvs"), 2)
    m = qvsim.apply_circuit(st, c, strategy="paired-cached")
    assert m["strategy"] == "paired-cached"
    amps = st.read_state()
    assert abs(amps[0] - 1 / math.sqrt(2)) <= 1e-15 and abs(amps[3] - 1 / math.sqrt(2)) <= 1e-15
    with pytest.raises(qvsim.QvsimError, match="unknown strategy"):
        qvsim.apply_circuit(st, c, strategy="gpux")
    if not cuda_present():
        with pytest.raises(qvsim.QvsimError, match="gpu strategy"):
            qvsim.apply_circuit(st, c, strategy="gpu")


@pytest.mark.gpu
def test_dropin_gpu_strategy_bit_equal_to_paired_cached(qvsim, tmp_path):
    cases = [qvsim.random_circuit(n, d, seed=s) for n, d, s in [(6, 40, 7), (10, 200, 3), (12, 300, 5), (16, 400, 9)]]
    cases.append(qvsim.parse_circuit("qubits 18\n" + "".join(f"h {q}\n" for q in range(18)) +
                                     "".join(f"cx {q} {q + 1}\nrz {q + 1} 0.3\n" for q in range(17))))
    for i, c in enumerate(cases):
        a = qvsim.StateStore.create(str(tmp_path / f"a{i}.qvs"), c.n_qubits)
        b = qvsim.StateStore.create(str(tmp_path / f"b{i}.qvs"), c.n_qubits)
        ma = qvsim.apply_circuit(a, c, strategy="gpu")
        qvsim.apply_circuit(b, c, strategy="paired-cached")
        assert ma["strategy"] == "gpu" and ma["gates_applied"] == len(c)
        assert a.read_state() == b.read_state(), i  # list equality: bit for bit (+-0 equal)
        assert abs(a.norm() - 1.0) <= 1e-12
    # the process really runs the B200 path: libqvg.so and the drop-in are mapped
    maps = open("/proc/self/maps").read()
    assert "libqvg.so" in maps and "libqvsim_gpu.so" in maps


@pytest.mark.gpu
def test_dropin_reference_smoke_cases_on_gpu(qvsim, tmp_path):
    """The reference's own Python smoke cases (proj/tests/python/test_smoke.py:
    Bell, GHZ, accumulation on an existing store) with strategy="gpu"."""
    st = qvsim.StateStore.create(str(tmp_path / "ghz.qvs"), 3)
    qvsim.apply_circuit(st, qvsim.parse_circuit("qubits 3\nh 0\ncx 0 1\ncx 1 2\n"), strategy="gpu")
    amps = st.read_state()
    r = 1 / math.sqrt(2)
    assert abs(amps[0] - r) <= 1e-12 and abs(amps[7] - r) <= 1e-12
    assert all(abs(a) <= 1e-12 for a in amps[1:7])
    top = qvsim.top_amplitudes(st, 2)
    assert sorted(i for i, _ in top) == [0, 7]
    # runs accumulate on the stored state (reference tools/qvsim_main.cpp:90-97)
    qvsim.apply_circuit(st, qvsim.parse_circuit("qubits 3\ncx 1 2\ncx 0 1\nh 0\n"), strategy="gpu")
    back = st.read_state()
    assert abs(back[0] - 1) <= 1e-12 and all(abs(a) <= 1e-12 for a in back[1:])
