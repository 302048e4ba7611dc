set -x
export QVG_JIT_VERBOSE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "jit" > gpurun_out/j_tests.log 2>&1; echo "jit tests rc=$?"; tail -15 gpurun_out/j_tests.log
timeout 1200 python tools/pass_times.py --n 30 --variants "jit=0;jit=2" > gpurun_out/jt_c128.json 2> gpurun_out/jt_c128.err; echo "pt rc=$?"; tail -8 gpurun_out/jt_c128.err
timeout 900 python tools/pass_times.py --n 30 --precision 64 --variants "jit=0;jit=2" > gpurun_out/jt_c64.json 2> gpurun_out/jt_c64.err; echo "pt64 rc=$?"; tail -8 gpurun_out/jt_c64.err
timeout 600 python tools/pass_times.py --n 26 --variants "jit=0;jit=2" --only config1_qft,config0_u3_ladder_l4 > gpurun_out/jt_c128_n26.json 2> gpurun_out/jt_c128_n26.err; echo "pt26 rc=$?"; tail -4 gpurun_out/jt_c128_n26.err
