set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q > gpurun_out/p_tests.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/p_tests.log
timeout 900 python tools/pipe_ab.py --n 30 --reps 3 > gpurun_out/pipe_ab_c128.json 2> gpurun_out/pipe_ab_c128.err; echo "ab rc=$?"; cat gpurun_out/pipe_ab_c128.err | tail -8
timeout 600 python tools/pipe_ab.py --n 30 --reps 3 --precision 64 > gpurun_out/pipe_ab_c64.json 2> gpurun_out/pipe_ab_c64.err; echo "ab64 rc=$?"; tail -6 gpurun_out/pipe_ab_c64.err
