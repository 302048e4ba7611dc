export QVG_SEGV_TRACE=1
timeout 600 python tools/jit_exit_probe.py torch graph > gpurun_out/probe.log 2>&1; echo "[probe] rc=$?"; tail -5 gpurun_out/probe.log
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/full2_tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/full2_tests.log
