#!/bin/bash
# A/B of the hot-table step kernel (GN_PART_HOT_KB) on C5 scale 24, one part
out=gpurun_out/${1:-r2hot}
mkdir -p $out
GN_PART_HOT_KB=64 timeout 900 python -m pytest tests/test_partition_gpu.py -q -x > $out/part_tests_hot.log 2>&1; echo "part tests hot rc=$?" >> $out/rc.txt
for kb in 0 1 16 64 128 192; do
  for dt in fp64; do
    GN_PART_HOT_KB=$kb timeout 600 python tools/probe_c5.py --dtype $dt --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
  done
done
