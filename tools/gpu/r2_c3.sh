set -x
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "config3" > gpurun_out/c3_tests.log 2>&1; echo "c3 rc=$?"; tail -5 gpurun_out/c3_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/pe_tests.log 2>&1; echo "pe rc=$?"; tail -5 gpurun_out/pe_tests.log
timeout 900 python tools/pass_times.py --n 30 --variants "jit=0;jit=1;jit=3" --reps 3 > gpurun_out/jab_c128.json 2> gpurun_out/jab_c128.err; echo "ab rc=$?"; grep config gpurun_out/jab_c128.err
timeout 900 python tools/pass_times.py --n 30 --precision 64 --variants "jit=0;jit=1" --reps 3 > gpurun_out/jab_c64.json 2> gpurun_out/jab_c64.err; echo "ab64 rc=$?"; grep config gpurun_out/jab_c64.err
