#!/bin/bash
out=gpurun_out/${1:-s6}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 600 python tools/probe_active.py > $out/active.json 2> $out/active.err; echo "active rc=$?" >> $out/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=8 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
cat $out/rc.txt; cat $out/active.json; tail -4 $out/pytest.log; cut -c1-400 $out/bench_c5.json
