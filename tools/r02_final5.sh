#!/bin/bash
# Closing validation of the round: smoke, the -m gpu suite, the default bench
# line (C5, one part) with its reference arm, and the other configs' lines.
out=gpurun_out/${1:-r2f5}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
nvidia-smi > $out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "bench ref rc=$?" >> $out/rc.txt
timeout 900 python bench.py --dtype fp32 --no-cpu-baseline > $out/bench_c5_fp32.json 2> $out/bench_c5_fp32.err; echo "bench c5 fp32 rc=$?" >> $out/rc.txt
for c in C2 C3 C4; do
  timeout 600 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c rc=$?" >> $out/rc.txt
done
cat $out/rc.txt
