#!/bin/bash
# A/B: degree threshold of the warp-split long rows (GN_PART_LONG)
out=gpurun_out/${1:-r2long}
mkdir -p $out
GN_PART_LONG=4096 timeout 900 python -m pytest tests/test_partition_gpu.py -q -x > $out/part_tests_long4096.log 2>&1; echo "part tests long4096 rc=$?" >> $out/rc.txt
for env in "GN_PART_LONG=1024" "GN_PART_LONG=2048" "GN_PART_LONG=4096" "GN_PART_LONG=8192" "GN_PART_LONG=16384" "GN_PART_LONG=65536"; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
GN_PART_LONG=4096 timeout 600 python tools/probe_c5.py --dtype fp32 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
