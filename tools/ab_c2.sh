mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in "GN_X=0" "GN_NO_ITEM_CACHE=1"; do
  echo "== $cfg"
  env $cfg python tools/probe.py --which C2,C3,C5S20 --grid 0 --iters 1000 --reps 2 --dtypes fp64,fp32 2>&1 | grep -v "^#\|gen\|create"
done
