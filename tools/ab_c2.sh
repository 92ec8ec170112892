mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for rep in 1 2; do
for lib in "" exp/libgnb200_old.so; do
  echo "== $lib"
  GN_LIB=$lib python tools/probe.py --which C2,C3,C5S20 --grid 0 --iters 1000 --reps 2 --dtypes fp64 2>&1 | grep -v "^#\|gen\|create" | cut -c1-100
done; done
