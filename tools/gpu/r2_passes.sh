set -x
timeout 600 python -m pytest tests/test_gpu_edges.py -q -k "warp_shuffle" > gpurun_out/p_low.log 2>&1; echo "low rc=$?"; tail -5 gpurun_out/p_low.log
timeout 900 python tools/pass_times.py --n 30 --pipes 0,4 > gpurun_out/pt_c128.json 2> gpurun_out/pt_c128.err; echo "pt rc=$?"; tail -6 gpurun_out/pt_c128.err
timeout 600 python tools/pass_times.py --n 30 --precision 64 --pipes 0,4 > gpurun_out/pt_c64.json 2> gpurun_out/pt_c64.err; echo "pt64 rc=$?"; tail -6 gpurun_out/pt_c64.err
M=gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__block_size,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:k_tile --csv --log-file gpurun_out/tma_ll_4.csv python tools/pass_profile.py --n 28 --circuit sweep --pipe 4 > gpurun_out/tma_ll_4.log 2>&1; echo "ll rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_tma -s 4 -c 1 -o gpurun_out/tma_full python tools/pass_profile.py --n 28 --circuit sweep --pipe 4 > gpurun_out/tma_full.log 2>&1; echo "full rc=$?"
