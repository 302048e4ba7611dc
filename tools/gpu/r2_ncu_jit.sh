set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qvg_jit -s 4 -c 1 -o gpurun_out/qftjit_full python tools/pass_profile.py --n 28 --circuit qft --jit 2 > gpurun_out/qftjit_full.log 2>&1; echo "qft rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qvg_jit -s 3 -c 1 -o gpurun_out/gridjit_full python tools/pass_profile.py --n 28 --circuit grid --jit 2 > gpurun_out/gridjit_full.log 2>&1; echo "grid rc=$?"
