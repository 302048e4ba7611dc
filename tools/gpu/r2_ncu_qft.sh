set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 4 -c 2 -o gpurun_out/qft_full python tools/pass_profile.py --n 28 --circuit qft --pipe 0 > gpurun_out/qft_full.log 2>&1; echo "qft rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -o gpurun_out/grid_full python tools/pass_profile.py --n 28 --circuit grid --pipe 0 > gpurun_out/grid_full.log 2>&1; echo "grid rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 5 -c 1 -o gpurun_out/sweepcx_full python tools/pass_profile.py --n 28 --circuit sweep --pipe 0 > gpurun_out/sweepcx_full.log 2>&1; echo "sweep rc=$?"
for g in 0 2; do timeout 300 python tools/small_ab.py --reps 20 --sizes 16,20,22 --graph $g > gpurun_out/small_ab_g$g.jsonl 2>&1; done
cat gpurun_out/small_ab_g0.jsonl gpurun_out/small_ab_g2.jsonl
