#!/bin/bash
out=gpurun_out/${1:-r2b}
mkdir -p $out
timeout 900 python -m pytest tests/test_partition_gpu.py tests/test_fuzz_gpu.py -q -x > $out/part_tests.log 2>&1; echo "part tests rc=$?" >> $out/rc.txt
for dt in fp64 fp32; do
  timeout 600 python tools/probe_c5.py --dtype $dt >> $out/probe.jsonl 2>> $out/probe.err
  GN_PART_BAND=0 timeout 600 python tools/probe_c5.py --dtype $dt >> $out/probe.jsonl 2>> $out/probe.err
done
for u in 8192 131072; do GN_BAND_UNIT=$u timeout 600 python tools/probe_c5.py --dtype fp64 >> $out/probe.jsonl 2>> $out/probe.err; done
GN_BAND_DIRECT=0 timeout 600 python tools/probe_c5.py --dtype fp64 >> $out/probe.jsonl 2>> $out/probe.err
echo done >> $out/rc.txt
