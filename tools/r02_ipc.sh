#!/bin/bash
# the 2-process IPC test on one GPU; ncu re-capture of the C5 step (LEX default)
out=gpurun_out/${1:-r2ipc}
mkdir -p $out
timeout 900 python -m pytest tests/test_ipc_gpu.py -q -x > $out/ipc.log 2>&1; echo "ipc rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s 0 -c 1 \
    -o $out/c5step python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/ncu.log 2>&1
echo "ncu step rc=$?" >> $out/rc.txt
