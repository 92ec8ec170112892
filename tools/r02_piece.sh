#!/bin/bash
out=gpurun_out/${1:-r2s}
mkdir -p $out
timeout 900 python -m pytest tests/test_partition_gpu.py -q -x > $out/part_tests.log 2>&1; echo "part tests rc=$?" >> $out/rc.txt
GN_PIECE_SORT=2 timeout 900 python -m pytest tests/test_partition_gpu.py -q -x > $out/part_tests_sort2.log 2>&1; echo "part tests sort2 rc=$?" >> $out/rc.txt
for env in "" "GN_PIECE_SORT=1" "GN_PIECE_SORT=2" "GN_PIECE_LEN=1024" "GN_PIECE_LEN=4096" "GN_PIECE_SORT=2 GN_PIECE_LEN=1024" "GN_PIECE_SORT=2 GN_PIECE_LEN=512"; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 >> $out/probe.jsonl 2>> $out/probe.err
done
