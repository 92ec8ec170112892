mkdir -p gpurun_out
for lib in "" exp/libgnb200_t768.so exp/libgnb200_t1024.so; do
  echo "== $lib"
  GN_LIB=$lib python tools/probe.py --which C2,C3,C5S20 --grid 0 --iters 1000 --reps 2 --dtypes fp64,fp32 2>&1 | grep -v "^#\|gen\|create" | cut -c1-130
done
