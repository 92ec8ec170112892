#!/bin/bash
# A/B: 16-bit delta chunk slices (GN_PART_DELTA)
out=gpurun_out/${1:-r2delta}
mkdir -p $out
timeout 1200 python -m pytest tests/test_partition_gpu.py -q -x > $out/part_tests.log 2>&1; echo "part tests rc=$?" >> $out/rc.txt
for env in "GN_PART_DELTA=0" "GN_PART_DELTA=1"; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
