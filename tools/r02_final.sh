#!/bin/bash
# Round-2 final measurement pass: smoke, the -m gpu suite, every bench line,
# the reference arm, the default bench's launch list, the scaling projection.
out=gpurun_out/${1:-r2final}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
nproc > $out/host.txt; nvidia-smi -L >> $out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --dtype fp32 --no-cpu-baseline > $out/bench_c5_fp32.json 2> $out/bench_c5_fp32.err; echo "bench c5 fp32 rc=$?" >> $out/rc.txt
for c in C2 C3 C4; do timeout 900 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c rc=$?" >> $out/rc.txt; done
timeout 900 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "bench ref rc=$?" >> $out/rc.txt
timeout 1200 python tools/probe_scaling.py --scale 24 --iters 30 > $out/scaling.json 2> $out/scaling.err; echo "scaling rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/launches.log 2>&1; echo "launches rc=$?" >> $out/rc.txt
