#!/bin/bash
# A/B: degree threshold of the warp-split long rows (GN_PART_LONG), piece length
out=gpurun_out/${1:-r2long}
mkdir -p $out
GN_PART_LONG=128 timeout 900 python -m pytest tests/test_partition_gpu.py -q -x > $out/part_tests_long128.log 2>&1; echo "part tests long128 rc=$?" >> $out/rc.txt
for env in "GN_PART_LONG=512" "GN_PART_LONG=256" "GN_PART_LONG=128" "GN_PART_LONG=64" "GN_PART_LONG=128 GN_PIECE_LEN=256" "GN_PART_LONG=1024"; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
