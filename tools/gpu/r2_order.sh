for k in "jit" "perm" "not jit and not perm"; do
  timeout 600 python -X faulthandler -m pytest tests/test_gpu_parity.py -q -x -k "$k" > gpurun_out/seg.log 2>&1; echo "[$k] rc=$?"; tail -4 gpurun_out/seg.log; grep -A12 "Fatal Python" gpurun_out/seg.log | head -20
done
timeout 900 python tools/pass_times.py --n 30 --variants "tile_order=0;tile_order=1;perm=0,tile_order=1" --reps 3 > gpurun_out/ord_c128.json 2> gpurun_out/ord_c128.err; echo "ab rc=$?"; grep config gpurun_out/ord_c128.err
