#!/bin/bash
# chunk/threshold sweep around the defaults (chunk 128, threshold 1024)
out=gpurun_out/${1:-r2chunk}
mkdir -p $out
for env in "GN_PART_LONG=1024" "GN_PART_LONG=512" "GN_PART_LONG=256" "GN_PART_CHUNK=96" "GN_PART_CHUNK=160" "GN_PART_LONG=512 GN_PART_CHUNK=192"; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
