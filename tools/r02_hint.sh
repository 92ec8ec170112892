#!/bin/bash
# A/B of the step kernel's cache policies (GN_PART_HINT builds) + the gather-ceiling microbenchmark
out=gpurun_out/${1:-r2h}
mkdir -p $out
timeout 300 exp/gather_ceiling > $out/ceiling.jsonl 2> $out/ceiling.err; echo "ceiling rc=$?" >> $out/rc.txt
for lib in "" exp/lib_h1.so exp/lib_h2.so exp/lib_h3.so; do
  for dt in fp64 fp32; do
    GN_LIB=$lib timeout 600 python tools/probe_c5.py --dtype $dt --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
  done
done
