export QVG_SEGV_TRACE=1
QVG_JIT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not jit and not perm" > gpurun_out/seg0.log 2>&1; echo "[jit off] rc=$?"; tail -3 gpurun_out/seg0.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not jit and not perm" > gpurun_out/seg1.log 2>&1; echo "[jit on] rc=$?"; tail -40 gpurun_out/seg1.log | grep -v "^\.\+"
