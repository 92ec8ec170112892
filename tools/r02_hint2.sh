#!/bin/bash
# A/B: L1 policy of the long rows' gathers (GN_PART_HINT 4 evict_first, 5 no_allocate)
out=gpurun_out/${1:-r2h2}
mkdir -p $out
for lib in "" exp/lib_h4.so exp/lib_h5.so; do
  for dt in fp64 fp32; do
    GN_LIB=$lib timeout 600 python tools/probe_c5.py --dtype $dt --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
  done
done
