set -x
nvidia-smi --query-gpu=name,memory.total,memory.free --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --deselect "tests/test_gpu_fullsize.py::test_n30_configs_match_reference_engine[config3_grid_5x6_c24_n30]" --durations=25 > gpurun_out/gpu1_tests.log 2>&1
echo "tests rc=$?"
tail -40 gpurun_out/gpu1_tests.log
