for cfg in "1 0" "1 4" "0 4"; do set -- $cfg
  QVG_JIT_SPLIT=$1 QVG_JIT_MINB=$2 timeout 900 python tools/pass_times.py --n 30 --variants "jit=0;jit=2" --reps 2 > gpurun_out/jt2_s$1_m$2.json 2> gpurun_out/jt2_s$1_m$2.err; echo "split=$1 minb=$2 rc=$?"; grep config gpurun_out/jt2_s$1_m$2.err
done
