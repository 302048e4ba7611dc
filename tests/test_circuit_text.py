"""Circuit text parser/serializer: differential against the reference's own
parse_circuit/serialize_circuit (reference circuit_io.cpp:68-202, driven
through oracle/_ref). Every input must give the same ops (bit for bit), the
same qubit count and the same serialization, or a ParseError on the same
line. The inputs restate the reference's grammar tests
(reference tests/test_circuit_io.cpp:28-200), plus a seeded mutation fuzz."""
import re

import numpy as np
import pytest

from oracle.oracle import RefEngine

pytestmark = pytest.mark.skipif(not RefEngine.available(), reason="oracle/_ref not built")

# (text, qubits override, strict)
CASES = [
    ("qubits 3\nh 0\nx 1\ny 2\nz 0\ns 1\nsdg 1\nt 2\ntdg 2\nrx 0 0.5\nry 1 -1.25\nrz 2 3.141592653589793\n"
     "u 0 0 0 1 0 1 0 0 0\ncx 0 2\ncz 2 1\n", None, False),
    ("# leading comment\n\n   qubits 2   \n\th 0 # trailing comment\n  \n#cx 0 1 whole-line comment\ncx 0 1\n\n",
     None, False),
    ("qubits 1\nh 0", None, False),
    ("qubits 4\nh 3\n", None, False),
    ("h 3\n", 4, False),
    ("qubits 4\nh 0\n", 4, False),
    ("qubits 4\nh 0\n", 5, False),
    ("h 0\n", None, False),
    ("", 3, False),
    ("h 0\nqubits 2\n", 2, False),
    ("qubits 2\nqubits 2\nh 0\n", None, False),
    ("qubits 0\nh 0\n", None, False),
    ("qubits -3\nh 0\n", None, False),
    ("qubits two\nh 0\n", None, False),
    ("qubits 2 2\nh 0\n", None, False),
    ("qubits\nh 0\n", None, False),
    ("qubits 2\nh 0\nfoo 1\n", None, False),
    ("qubits 2\nh\n", None, False),
    ("qubits 2\nh 0 1\n", None, False),
    ("qubits 2\nrx 0\n", None, False),
    ("qubits 2\nrx 0 a\n", None, False),
    ("qubits 2\nrx 0 nan\n", None, False),
    ("qubits 2\nrx 0 inf\n", None, False),
    ("qubits 2\nh -1\n", None, False),
    ("qubits 2\nh 1.5\n", None, False),
    ("qubits 2\ncx 0\n", None, False),
    ("qubits 2\nu 0 1 0 0 0 0 0 1\n", None, False),
    ("qubits 2\nh 0\nh 2\n", None, False),
    ("qubits 2\ncx 0 2\n", None, False),
    ("qubits 2\ncx 2 0\n", None, False),
    ("h 0\nh 5\n", 3, False),
    ("qubits 2\ncx 1 1\n", None, False),
    ("qubits 2\ncz 0 0\n", None, False),
    ("qubits 1\nu 0 0.70710678 0 0.70710678 0 0.70710678 0 -0.70710678 0\n", None, False),
    ("qubits 1\nu 0 0.70710678 0 0.70710678 0 0.70710678 0 -0.70710678 0\n", None, True),
    ("qubits 1\nu 0 1 0 0 0 0 0 2 0\n", None, False),
    ("qubits 1\nrz 0 0.30000000000000004\n", None, False),
    ("qubits 2\nrx 0 1e-3\nry 1 -0.0\nrz 0 +2.5\n", None, False),
    ("qubits 2\nRX 0 1\n", None, False),
    ("qubits 3\ncx 0 1 2\n", None, False),
    ("qubits 3\ncz 2\n", None, False),
]


def ours(qv, text, qubits, strict):
    try:
        c = qv.parse_circuit(text, qubits, strict)
    except qv.ParseError as e:
        m = re.match(r"line (\d+):", str(e))
        return ("ParseError", int(m.group(1)) if m else -1)
    return c.n_qubits, c.gates(), c.to_text()


def same(qv, ref, text, qubits, strict):
    a, b = ours(qv, text, qubits, strict), ref.parse(text, qubits, strict)
    if isinstance(b[0], str) or isinstance(a[0], str):
        assert a == b, (text, qubits, strict, a, b)
        return a[0] != "ParseError"
    assert a[0] == b[0], text
    assert a[1].tobytes() == b[1].tobytes(), text
    assert a[2] == b[2], text
    return True


@pytest.mark.parametrize("i", range(len(CASES)))
def test_parser_matches_reference(qv, i):
    same(qv, RefEngine(), *CASES[i])


def test_random_circuit_text_matches_reference(qv):
    """reference tests/test_circuit_io.cpp:189-200: random circuits through
    text, both implementations."""
    ref = RefEngine()
    rng = np.random.default_rng(7)
    for _ in range(100):
        n, depth, seed = int(rng.integers(1, 11)), int(rng.integers(1, 41)), int(rng.integers(1 << 62))
        ops, text = ref.random_circuit(n, depth, seed)
        c = qv.random_circuit(n, depth, seed)
        assert c.to_text() == text
        assert same(qv, ref, text, None, False)


def test_mutation_fuzz_matches_reference(qv):
    """Seeded token-level mutations of valid circuit text: drop, duplicate or
    replace one token, or join two lines. Ours and the reference must agree
    on every outcome (ops or the error line)."""
    ref = RefEngine()
    rng = np.random.default_rng(2508)
    junk = ["0", "1", "7", "-1", "1.5", "nan", "x", "cx", "qubits", "#", "1e309", "0x10", "", "u"]
    agreed_ok = agreed_err = 0
    for trial in range(400):
        _, text = ref.random_circuit(int(rng.integers(1, 6)), int(rng.integers(1, 8)), trial)
        lines = text.splitlines()
        li = int(rng.integers(len(lines)))
        toks = lines[li].split(" ")
        ti = int(rng.integers(len(toks)))
        op = int(rng.integers(4))
        if op == 0 and len(toks) > 1:
            del toks[ti]
        elif op == 1:
            toks.insert(ti, toks[ti])
        elif op == 2:
            toks[ti] = junk[int(rng.integers(len(junk)))]
        elif li + 1 < len(lines):
            lines[li + 1] = lines[li] + " " + lines[li + 1]
        lines[li] = " ".join(toks)
        mutated = "\n".join(lines) + ("\n" if rng.integers(2) else "")
        if same(qv, ref, mutated, None, bool(rng.integers(2))):
            agreed_ok += 1
        else:
            agreed_err += 1
    assert agreed_ok > 20 and agreed_err > 100
