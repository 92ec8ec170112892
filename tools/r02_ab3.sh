#!/bin/bash
# A/B on C5 scale 24 one part fp64 (adaptive long threshold): LEX=3, unroll builds
out=gpurun_out/${1:-r2ab3}
mkdir -p $out
for env in "GN_PART_LEX=1" "GN_PART_LEX=3" "GN_LIB=exp/lib_u12.so" "GN_LIB=exp/lib_u16.so" "GN_LIB=exp/lib_u16m3.so"; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
