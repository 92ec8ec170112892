#!/bin/bash
out=gpurun_out/${1:-r2n}
mkdir -p $out
python tools/probe_c5.py --reps 1 --iters 20 > $out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_part_step|k_part_probe|k_part_long_combine" -s 0 -c 18 \
    -o $out/c5probe python tools/probe_c5.py --reps 1 --iters 20 > $out/ncu.log 2>&1
echo "rc=$?" >> $out/ncu.log
