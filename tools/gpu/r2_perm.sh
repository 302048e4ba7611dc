set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/pp_tests.log 2>&1; echo "pe rc=$?"; tail -15 gpurun_out/pp_tests.log
timeout 900 python tools/pass_times.py --n 30 --variants "perm=0;perm=1" --reps 3 > gpurun_out/perm_c128.json 2> gpurun_out/perm_c128.err; echo "ab rc=$?"; grep config gpurun_out/perm_c128.err
timeout 900 python tools/pass_times.py --n 30 --precision 64 --variants "perm=0;perm=1" --reps 3 > gpurun_out/perm_c64.json 2> gpurun_out/perm_c64.err; echo "ab64 rc=$?"; grep config gpurun_out/perm_c64.err
