#!/bin/bash
out=gpurun_out/${1:-r2b3}
mkdir -p $out
timeout 900 python -m pytest tests/test_partition_gpu.py tests/test_fuzz_gpu.py -q -x > $out/part_tests.log 2>&1; echo "part tests rc=$?" >> $out/rc.txt
for dt in fp64 fp32; do
  timeout 600 python tools/probe_c5.py --dtype $dt >> $out/probe.jsonl 2>> $out/probe.err
done
python tools/probe_c5.py --reps 1 --iters 20 > $out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_part_band|k_part_long_combine" -s 0 -c 2 \
    -o $out/band python tools/probe_c5.py --reps 1 --iters 20 > $out/ncu.log 2>&1
echo "ncu rc=$?" >> $out/rc.txt
