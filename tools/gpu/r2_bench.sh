set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/f_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo "ref rc=$?"; cat gpurun_out/f_bench_ref.json
timeout 1500 python bench.py --configs > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err; echo "configs rc=$?"; cat gpurun_out/f_configs.jsonl | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 30 -c 120 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-config4 > gpurun_out/f_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/f_launches.csv --skip 30 --out gpurun_out/f_bench_launches.json; echo "sum rc=$?"
