set -x
timeout 1500 python -m pytest tests -m gpu -x -q --deselect "tests/test_gpu_fullsize.py::test_n30_configs_match_reference_engine[config3_grid_5x6_c24_n30]" --durations=15 > gpurun_out/r2_tests.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/r2_tests.log
for g in 0 2; do timeout 300 python tools/small_ab.py --reps 20 --sizes 16,20,22 --graph $g > gpurun_out/small_ab_g$g.jsonl 2>&1; done
cat gpurun_out/small_ab_g0.jsonl gpurun_out/small_ab_g2.jsonl
