#!/bin/bash
# Round-end measurement pass on the GPU box (run through gpurun); outputs in gpurun_out/m/.
M=gpurun_out/m
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
# launch list of the default bench (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $M/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $M/ncu_launches.log 2>&1; echo "launches rc=$?"
F="timeout 900 ncu --set full --clock-control none --import-source on -c 1"
$F -k regex:k_gn_loop -o $M/c2_loop python tools/probe.py --which C2 --grid 0 --iters 1000 --reps 1 --dtypes fp64 > $M/ncu_c2.log 2>&1; echo "c2 rc=$?"
$F -k regex:k_gn_loop -o $M/c3_loop python tools/probe.py --which C3 --grid 0 --iters 1000 --reps 1 > $M/ncu_c3.log 2>&1; echo "c3 rc=$?"
$F -k regex:k_gn_batch -o $M/c4_batch python tools/probe_batch.py 1024 fp32 > $M/ncu_c4.log 2>&1; echo "c4 rc=$?"
$F -k regex:k_gn_loop -o $M/c5_loop python tools/probe.py --which C5S24 --grid 0 --iters 5 --reps 1 > $M/ncu_c5.log 2>&1; echo "c5 rc=$?"
uptime >> $M/host_uptime.txt
