# one GPU: the -m gpu tests that changed + a short bench (ours) + the reference arm
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q -k "hooks or dropin or timing" > gpurun_out/b_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/b_tests.log
timeout 900 python bench.py --steps 8 --warmup 3 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_ours.json; tail -20 gpurun_out/bench_ours.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
cat gpurun_out/bench_ref.json; tail -5 gpurun_out/bench_ref.err
nproc; free -g | head -2
