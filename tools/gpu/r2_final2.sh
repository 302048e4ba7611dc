# follow-up of r2_final.sh: the new counter-law tests, per-pass ncu metrics (launch-skip counts matching kernels only), 6 CTAs/SM A/B
set -x
timeout 600 python -m pytest tests -m gpu -q -k "counter_law or load_ahead" > gpurun_out/f2_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/f2_tests.log
QVG_PKG_ROOT=$PWD/.variants/minb6 timeout 600 python tools/pass_times.py --variants "pipe=-1;pipe=5" --reps 3 > gpurun_out/minb6.json 2> gpurun_out/minb6.err; grep ^config gpurun_out/minb6.err
timeout 600 python tools/pass_times.py --variants "pipe=-1;pipe=5" --reps 3 > gpurun_out/minb5.json 2> gpurun_out/minb5.err; grep ^config gpurun_out/minb5.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in grid sweep qft ladder; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_tile --csv --log-file gpurun_out/f_pass_$c.csv python tools/pass_profile.py --n 30 --circuit $c > gpurun_out/f_pass_$c.log 2>&1; echo "pass $c rc=$?"
done
python tools/fused_ncu_summary.py C3_grid=gpurun_out/f_pass_grid.csv C2_sweep=gpurun_out/f_pass_sweep.csv C1_qft=gpurun_out/f_pass_qft.csv C0_ladder=gpurun_out/f_pass_ladder.csv > gpurun_out/f_fused_passes.json; echo "fsum rc=$?"
