#!/bin/bash
# new fuzz/partition tests; ncu --set full capture of the current C5 step (for ncu_summary.json)
out=gpurun_out/${1:-r2nf}
mkdir -p $out
timeout 1500 python -m pytest tests/test_fuzz_gpu.py tests/test_partition_gpu.py -q -x > $out/tests.log 2>&1; echo "tests rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s 0 -c 1 \
    -o $out/c5step python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/ncu.log 2>&1
echo "ncu step rc=$?" >> $out/rc.txt
