mkdir -p gpurun_out
for cfg in "GN_X=0" "GN_L2_PERSIST=60" "GN_L2_PERSIST=90"; do
  echo "== $cfg"
  env $cfg python tools/probe.py --which C5S24,C3 --grid 0 --iters 100 --reps 2 --dtypes fp32 2>&1 | grep -v "^#\|gen\|create"
done
