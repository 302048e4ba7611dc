# same-box A/B: the main build against a variant package built under .variants/<name> (copy paper_2508_15545_b200 + include there,
# make with EXTRA_NVFLAGS or edited sources; pass_times.py imports it through QVG_PKG_ROOT), two interleaved rounds.
#   bash tools/gpu/r2_variant_ab.sh <name>
for i in 1 2; do
for v in main variant; do
  if [ $v = variant ]; then export QVG_PKG_ROOT=$PWD/.variants/$1; else unset QVG_PKG_ROOT; fi
  echo "== $v"
  python tools/pass_times.py --variants "pipe=-1" --reps 3 2>&1 >/dev/null | grep ^config
done; done
