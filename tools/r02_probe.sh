#!/bin/bash
out=gpurun_out/${1:-r2p}
mkdir -p $out
timeout 600 python -m pytest tests/test_dropin_reference_gpu.py -q -x > $out/dropin.log 2>&1; echo "dropin rc=$?" >> $out/rc.txt
for lib in "" exp/lib_minb4.so exp/lib_u16.so exp/lib_minb4u16.so; do
  for dt in fp32 fp64; do
    GN_LIB=$lib timeout 600 python tools/probe_c5.py --dtype $dt >> $out/probe.jsonl 2>> $out/probe.err
  done
done
timeout 900 python bench.py --dtype fp64 --steps 3 --no-cpu-baseline > $out/bench_c5_fp64.json 2> $out/bench_c5_fp64.err
