export QVG_SEGV_TRACE=1
for m in "graph" "torch graph" "torch graph drain" "torch graph keep" "torch graph drain keep"; do timeout 120 python tools/jit_exit_probe.py $m > gpurun_out/probe.log 2>&1; echo "[$m] rc=$?"; tail -12 gpurun_out/probe.log; done
