M=gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__registers_per_thread,launch__grid_size,launch__block_size
for p in 0 2; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_tile --csv --log-file gpurun_out/pipe_ll_$p.csv python tools/pass_profile.py --n 28 --circuit sweep --pipe $p > gpurun_out/pipe_ll_$p.log 2>&1; echo "ll $p rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_pipe -s 1 -c 2 -o gpurun_out/pipe_full python tools/pass_profile.py --n 28 --circuit sweep --pipe 2 > gpurun_out/pipe_full.log 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 1 -c 2 -o gpurun_out/tile_full python tools/pass_profile.py --n 28 --circuit sweep --pipe 0 > gpurun_out/tile_full.log 2>&1; echo "full0 rc=$?"
