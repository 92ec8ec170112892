#!/bin/bash
# Full -m gpu suite, smoke, default bench (C5 partitioned N=1), C5 fp32, ncu of the step, scaling projection
out=gpurun_out/${1:-r2f}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=12 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --dtype fp32 --no-cpu-baseline > $out/bench_c5_fp32.json 2> $out/bench_c5_fp32.err; echo "bench c5 fp32 rc=$?" >> $out/rc.txt
timeout 1200 python tools/probe_scaling.py --scale 24 --iters 30 > $out/scaling.json 2> $out/scaling.err; echo "scaling rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s 0 -c 1 \
    -o $out/c5step python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/ncu.log 2>&1
echo "ncu step rc=$?" >> $out/rc.txt
