# same-box A/B: main build against a variant package under .variants/<name> (QVG_PKG_ROOT), two interleaved rounds
for i in 1 2; do
for v in main variant; do
  if [ $v = variant ]; then export QVG_PKG_ROOT=$PWD/.variants/$1; else unset QVG_PKG_ROOT; fi
  echo "== $v"
  python tools/pass_times.py --variants "pipe=-1" --reps 3 2>&1 >/dev/null | grep ^config
done; done
