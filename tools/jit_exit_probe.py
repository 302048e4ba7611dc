"""Process-exit probe for the async JIT compile workers: apply circuits whose
passes queue JIT compiles, then exit. Flags: torch (import torch first),
graph (apply each list 3x so CUDA graphs capture JIT kernels), drain (wait for
the compile queue), keep (states alive at exit). Prints 'exit ok'."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
flags = set(sys.argv[1:])
if "torch" in flags:
    import torch  # noqa: F401
import paper_2508_15545_b200 as qv  # noqa: E402

states = []
for n, prec in ((12, 128), (13, 64), (14, 128)):
    st = qv.StateVector.create(n, prec, 0)
    c = qv.qft_circuit(n, 1)[0]
    for _ in range(3 if "graph" in flags else 1):
        st.init_basis(0)
        qv.apply_circuit(st, c)
        if "drain" in flags:
            qv.jit_info(True)
    st.sync()
    print(n, prec, st.stats()["jit_passes"], st.stats()["graph_replays"], flush=True)
    if "keep" in flags:
        states.append(st)
print("exit ok", sorted(flags), flush=True)
