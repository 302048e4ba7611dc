# one GPU: the whole -m gpu suite (config-3 fixture pending), the default bench, the reference arm, the TMA tile A/B
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 2400 python -m pytest tests -m gpu -q --deselect "tests/test_gpu_fullsize.py::test_n30_configs_match_reference_engine[config3_grid_5x6_c24_n30]" --durations=30 > gpurun_out/m_tests.log 2>&1; echo "tests rc=$?"; tail -45 gpurun_out/m_tests.log
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/m_bench.json; tail -20 gpurun_out/m_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/m_bench_ref.json 2> gpurun_out/m_bench_ref.err; echo "ref rc=$?"
cat gpurun_out/m_bench_ref.json; tail -5 gpurun_out/m_bench_ref.err
timeout 900 python tools/pipe_ab.py --n 30 --reps 3 --pipes 0,4 > gpurun_out/tma_ab_c128.json 2> gpurun_out/tma_ab_c128.err; echo "ab rc=$?"; tail -8 gpurun_out/tma_ab_c128.err
