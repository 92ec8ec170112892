#!/bin/bash
# Full -m gpu suite, smoke, and the default bench line (C5 partitioned, N=1)
out=gpurun_out/${1:-r2f}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=12 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
