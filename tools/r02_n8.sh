#!/bin/bash
# per-kernel launch list of one part of the 8-way C5 partition (part 7) on one GPU
out=gpurun_out/${1:-r2n8}
mkdir -p $out
timeout 900 python tools/probe_scaling.py --gpus 8 --parts 7 --iters 20 > $out/plain.json 2> $out/plain.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python tools/probe_scaling.py --gpus 8 --parts 7 --iters 20 > $out/ncu.log 2>&1
echo "rc=$?" >> $out/rc.txt
