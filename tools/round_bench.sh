#!/bin/bash
# Round-end bench lines on the GPU box (run through gpurun); outputs in gpurun_out/m/.
M=gpurun_out/m
mkdir -p $M
run() { local name=$1; shift; "$@" > $M/$name.json 2> $M/$name.err; echo "$name rc=$?"; }
nproc > $M/host_nproc.txt; uptime > $M/host_uptime.txt
run bench_c2 python bench.py
run bench_c2_reference python bench.py --impl reference
run bench_c3 python bench.py --config C3 --no-cpu-baseline
run bench_c4 python bench.py --config C4 --no-cpu-baseline
run bench_c5 python bench.py --config C5 --no-cpu-baseline --steps 3 --warmup 3
run bench_c2_x16 python bench.py --starts 16 --no-cpu-baseline
run bench_c3_x16 python bench.py --config C3 --starts 16 --no-cpu-baseline
uptime >> $M/host_uptime.txt
