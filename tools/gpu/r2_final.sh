# Round-2 closing run on one B200: the whole -m gpu suite, the bench (ours + reference arm + per-config lines),
# the bench's ncu launch list, per-pass ncu metrics of the four fused BASELINE circuits, and one full ncu
# capture of a light grid pass on the load-ahead kernel.
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/f_tests.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/f_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo "ref rc=$?"; cat gpurun_out/f_bench_ref.json
timeout 1500 python bench.py --configs > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err; echo "configs rc=$?"; cut -c1-300 gpurun_out/f_configs.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 30 -c 120 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-config4 > gpurun_out/f_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/f_launches.csv --skip 30 --out gpurun_out/f_bench_launches.json; echo "sum rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in grid sweep qft ladder; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_tile --csv --log-file gpurun_out/f_pass_$c.csv python tools/pass_profile.py --n 30 --circuit $c > gpurun_out/f_pass_$c.log 2>&1; echo "pass $c rc=$?"
done
python tools/fused_ncu_summary.py C3_grid=gpurun_out/f_pass_grid.csv C2_sweep=gpurun_out/f_pass_sweep.csv C1_qft=gpurun_out/f_pass_qft.csv C0_ladder=gpurun_out/f_pass_ladder.csv > gpurun_out/f_fused_passes.json; echo "fsum rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_ahead -s 1 -c 1 -o gpurun_out/f_ahead_full python tools/pass_profile.py --n 28 --circuit grid > gpurun_out/f_ahead_full.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/f_ahead_full.ncu-rep --page raw --csv > gpurun_out/f_ahead_full_raw.csv 2>/dev/null; echo "raw rc=$?"
rm -f gpurun_out/f_ahead_full.ncu-rep.tmp
