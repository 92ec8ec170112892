#!/bin/bash
# quick A/B: partition GPU tests, C5 probe (fp32, fp64), a short default bench
out=gpurun_out/${1:-r2q}
mkdir -p $out
timeout 900 python -m pytest tests/test_partition_gpu.py tests/test_fuzz_gpu.py -q -x > $out/part_tests.log 2>&1; echo "part tests rc=$?" >> $out/rc.txt
for dt in fp32 fp64; do timeout 600 python tools/probe_c5.py --dtype $dt >> $out/probe.jsonl 2>> $out/probe.err; done
GN_BENCH_VERBOSE=1 timeout 900 python bench.py --steps 3 --no-cpu-baseline > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench rc=$?" >> $out/rc.txt
