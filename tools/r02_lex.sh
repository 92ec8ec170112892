#!/bin/bash
# A/B of the partitioned engine's row numbering (GN_PART_LEX, GN_PART_WINDOW) on C5 scale 24, one part
out=gpurun_out/${1:-r2lex}
mkdir -p $out
for env in "GN_PART_LEX=1 GN_PART_WINDOW=0" "GN_PART_LEX=2 GN_PART_WINDOW=0" "GN_PART_LEX=2" ; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
