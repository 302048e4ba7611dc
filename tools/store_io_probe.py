"""Raw QVSV file read throughput through StateStore.read_state (n=30 file in
/dev/shm) and the Kahan norm.

    python tools/store_io_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_15545_b200 as qv
n = 30
path = f"/dev/shm/iot-{os.getpid()}.qvs"
qv.StateStore.create(path, n, overwrite=True)
s = qv.StateStore.open(path)
for rep in range(3):
    t0 = time.perf_counter(); a = s.read_state(); t1 = time.perf_counter()
    print("read_state 16 GiB", round(t1 - t0, 3), "s", round((16 << 30) / (t1 - t0) / 1e9, 1), "GB/s", flush=True)
    del a
# write path via apply with empty circuit? use norm (read) as second probe
t0 = time.perf_counter(); s.norm(); print("norm", round(time.perf_counter() - t0, 3), flush=True)
os.remove(path)
