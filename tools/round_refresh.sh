#!/bin/bash
# Bench lines only (kernels unchanged since the last ncu pass); outputs in gpurun_out/m3/.
M=gpurun_out/m3
mkdir -p $M
run() { local name=$1; shift; timeout 1200 "$@" > $M/$name.json 2> $M/$name.err; echo "$name rc=$?"; }
nproc > $M/host_nproc.txt; uptime > $M/host_uptime.txt
run bench_c2 python bench.py
run bench_c2_reference python bench.py --impl reference
run bench_c3 python bench.py --config C3
run bench_c4 python bench.py --config C4
run bench_c5 python bench.py --config C5 --steps 3 --warmup 3
run bench_c5_part python bench.py --config C5 --partition --no-cpu-baseline --steps 3 --warmup 3
run bench_c2_x16 python bench.py --starts 16 --no-cpu-baseline
run bench_c3_x16 python bench.py --config C3 --starts 16 --no-cpu-baseline
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $M/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $M/ncu_launches.log 2>&1; echo "launches rc=$?"
uptime >> $M/host_uptime.txt
