for i in 1 2; do
for v in head lean; do
  if [ $v = head ]; then export QVG_PKG_ROOT=$PWD/.variants/head; else unset QVG_PKG_ROOT; fi
  echo "== $v"
  python tools/pass_times.py --variants "pipe=0" --reps 3 2>&1 >/dev/null | grep ^config
  python tools/pass_times.py --precision 64 --variants "pipe=0" --reps 3 2>&1 >/dev/null | grep ^config
  python tools/pass_times.py --n 26 --variants "pipe=-1" --reps 5 2>&1 >/dev/null | grep ^config
  python tools/pass_times.py --n 22 --variants "pipe=-1" --reps 5 2>&1 >/dev/null | grep ^config
done; done
