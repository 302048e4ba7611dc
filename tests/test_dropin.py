"""The reference-side drop-in (VERDICT r1 "missing" #3):
the reference's OWN engine and pybind11 module, rebuilt from copies of its
engine.hpp / engine.cpp with the `Strategy::gpu` branch added
(integration/reference_patch.py, integration/gpu_strategy.cpp, `make -C
oracle dropin`) and linked with libqvg.so. `qvsim.apply_circuit(store, c,
strategy="gpu")` — the reference's binding forwarding the tag to its C++
`apply_circuit(BlockStore&, ...)` — must equal the reference's own
paired-cached engine on the same QVSV file bit for bit.

Each case runs in a fresh interpreter: the reference's module and this
package's both bind C++ types named qvsim::Circuit etc., which pybind11 does
not allow in one process."""
import os
import subprocess
import sys
import textwrap

import pytest

from conftest import ROOT

DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin", "python")


def run_isolated(body, tmp_path):
    if not os.path.isdir(os.path.join(DROPIN, "qvsim")):
        pytest.fail("reference drop-in not built: make -C oracle dropin (needs /root/reference once)")
    code = textwrap.dedent("""
        import math, os, sys
        try:  # torch before any CUDA library of ours: on a box without a driver, torch's import
            import torch  # noqa: F401  segfaults once libcudart is already mapped
        except Exception:
            pass
        sys.path.insert(0, {dropin!r})
        import qvsim
        assert qvsim.__file__.startswith({dropin!r}), qvsim.__file__
        tmp = {tmp!r}
        def cuda_present():
            try:
                import torch
                return torch.cuda.is_available()
            except Exception:
                return False
    """).format(dropin=DROPIN, tmp=str(tmp_path)) + textwrap.dedent(body)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r.stdout


def test_dropin_module_is_the_reference_with_a_gpu_tag(tmp_path):
    """CPU: the rebuilt reference module runs its own strategies, knows the
    "gpu" tag, and (without a device) fails it loudly as QvsimError."""
    run_isolated("""
        c = qvsim.parse_circuit("qubits 2\\nh 0\\ncx 0 1\\n")
        st = qvsim.StateStore.create(os.path.join(tmp, "bell.qvs"), 2)
        m = qvsim.apply_circuit(st, c, strategy="paired-cached")
        assert m["strategy"] == "paired-cached"
        amps = st.read_state()
        assert abs(amps[0] - 1 / math.sqrt(2)) <= 1e-15 and abs(amps[3] - 1 / math.sqrt(2)) <= 1e-15
        try:
            qvsim.apply_circuit(st, c, strategy="gpux")
            raise SystemExit("unknown tag accepted")
        except qvsim.QvsimError as e:
            assert "unknown strategy" in str(e)
        if not cuda_present():
            try:
                qvsim.apply_circuit(st, c, strategy="gpu")
                raise SystemExit("gpu strategy ran without a device")
            except qvsim.QvsimError as e:
                assert "gpu strategy" in str(e)
    """, tmp_path)


@pytest.mark.gpu
def test_dropin_gpu_strategy_bit_equal_to_paired_cached(tmp_path):
    out = run_isolated("""
        cases = [qvsim.random_circuit(n, d, seed=s) for n, d, s in [(6, 40, 7), (10, 200, 3), (12, 300, 5),
                                                                  (16, 400, 9)]]
        cases.append(qvsim.parse_circuit("qubits 18\\n" + "".join(f"h {q}\\n" for q in range(18)) +
                                         "".join(f"cx {q} {q + 1}\\nrz {q + 1} 0.3\\n" for q in range(17))))
        for i, c in enumerate(cases):
            a = qvsim.StateStore.create(os.path.join(tmp, f"a{i}.qvs"), c.n_qubits)
            b = qvsim.StateStore.create(os.path.join(tmp, f"b{i}.qvs"), c.n_qubits)
            ma = qvsim.apply_circuit(a, c, strategy="gpu")
            qvsim.apply_circuit(b, c, strategy="paired-cached")
            assert ma["strategy"] == "gpu" and ma["gates_applied"] == len(c), ma
            assert a.read_state() == b.read_state(), i  # list equality: bit for bit (+-0 equal)
            assert abs(a.norm() - 1.0) <= 1e-12
        # the process really ran the B200 path: libqvg.so and the drop-in are mapped
        maps = open("/proc/self/maps").read()
        assert "libqvg.so" in maps and "libqvsim_gpu.so" in maps
        print("dropin ok", len(cases))
    """, tmp_path)
    assert "dropin ok 5" in out


@pytest.mark.gpu
def test_dropin_reference_smoke_cases_on_gpu(tmp_path):
    """The reference's own Python smoke cases (proj/tests/python/test_smoke.py:
    GHZ, top amplitudes, accumulation on an existing store) with strategy="gpu"."""
    run_isolated("""
        st = qvsim.StateStore.create(os.path.join(tmp, "ghz.qvs"), 3)
        qvsim.apply_circuit(st, qvsim.parse_circuit("qubits 3\\nh 0\\ncx 0 1\\ncx 1 2\\n"), strategy="gpu")
        amps = st.read_state()
        r = 1 / math.sqrt(2)
        assert abs(amps[0] - r) <= 1e-12 and abs(amps[7] - r) <= 1e-12
        assert all(abs(a) <= 1e-12 for a in amps[1:7])
        assert sorted(i for i, _ in qvsim.top_amplitudes(st, 2)) == [0, 7]
        # runs accumulate on the stored state (reference tools/qvsim_main.cpp:90-97)
        qvsim.apply_circuit(st, qvsim.parse_circuit("qubits 3\\ncx 1 2\\ncx 0 1\\nh 0\\n"), strategy="gpu")
        back = st.read_state()
        assert abs(back[0] - 1) <= 1e-12 and all(abs(a) <= 1e-12 for a in back[1:])
    """, tmp_path)
