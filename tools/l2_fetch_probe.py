"""Per-gate pass times at n = 30 complex128 for gates whose control / target
is a low qubit (32/64-B runs of touched amplitudes), after setting
cudaLimitMaxL2FetchGranularity from the environment (QVG_L2_FETCH=32|64|128;
the default is 64). Result (profiles/r02_l2_fetch.jsonl): no change, CX with
control qubit 1 or 2 stays at 3.95 ms (DRAM reads whole 128-B granules there).

    QVG_L2_FETCH=32 python tools/l2_fetch_probe.py
"""
import ctypes
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2508_15545_b200 as qv
if os.environ.get("QVG_L2_FETCH"):
    rt = ctypes.CDLL("libcudart.so.12")
    torch.cuda.init()
    rt.cudaDeviceSetLimit(0x05, ctypes.c_size_t(int(os.environ["QVG_L2_FETCH"])))  # cudaLimitMaxL2FetchGranularity
n=30
st=qv.StateVector.create(n,128,0)
st.set_option(qv.OPT_FUSE,0); st.set_option(qv.OPT_GRAPH,0)
c=qv.parse_circuit(f"qubits {n}\nh 0\n")
stream=torch.cuda.ExternalStream(st.stream())
def t(text):
    g=qv.parse_circuit(f"qubits {n}\n{text}\n").gates()
    st.apply_gates(g); st.sync()
    ms=[]
    for _ in range(5):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(stream); st.apply_gates(g,sync=False); e1.record(stream); st.sync(); ms.append(e0.elapsed_time(e1))
    return round(sorted(ms)[2],3)
out={k:t(k) for k in ("h 0","h 7","h 29","cx 0 1","cx 1 0","cx 1 16","cx 2 3","cx 2 17","cx 3 18","cx 4 19","cx 15 0","cz 1 9","cz 2 9","t 1","t 2","t 3")}
print(json.dumps(out))
