#!/bin/bash
# one iteration of the C5 work: partition tests, probes (default + knobs), the default bench line, then the full-budget tests
out=gpurun_out/${1:-r2i}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 900 python -m pytest tests/test_partition_gpu.py tests/test_fuzz_gpu.py tests/test_dropin_reference_gpu.py -q -x > $out/tests_a.log 2>&1; echo "tests a rc=$?" >> $out/rc.txt
for env in "" "GN_PART_INTERLEAVE=0" ${PROBE_ENVS}; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 >> $out/probe.jsonl 2>> $out/probe.err
done
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench rc=$?" >> $out/rc.txt
timeout 1500 python -m pytest tests/test_fullbudget_gpu.py -q -x --durations=0 > $out/tests_full.log 2>&1; echo "tests full rc=$?" >> $out/rc.txt
