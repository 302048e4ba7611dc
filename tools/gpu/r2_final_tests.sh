set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -22 gpurun_out/final_tests.log
