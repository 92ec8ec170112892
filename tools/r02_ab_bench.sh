#!/bin/bash
# A/B of the whole C5 pursuit (certificates on, the default bench line) under
# environment settings: one bench line per setting.
#   tools/r02_ab_bench.sh OUT "GN_PART_SPW=8" "GN_PART_LONG=512" ...
out=gpurun_out/${1:-r2abb}
shift
mkdir -p $out
for env in "" "$@"; do
  echo "{\"env\": \"$env\"}" >> $out/bench.jsonl
  env $env timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-certificate-report >> $out/bench.jsonl 2>> $out/bench.err
done
