mkdir -p gpurun_out
for cfg in "GN_X=0" "GN_GLOBAL_SORT=1"; do
  echo "== $cfg"
  env $cfg python tools/probe.py --which C5S24,C5S20,C3 --grid 0 --iters 100 --reps 2 --dtypes fp32 2>&1 | grep -v "^#\|gen\|create"
done
