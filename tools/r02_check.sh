#!/bin/bash
# Round-2 GPU check: smoke, the -m gpu suite, the default bench line (C5
# partitioned), C2, and the reference arm.  Outputs under gpurun_out/$1.
out=gpurun_out/${1:-r2}
mkdir -p $out
nproc > $out/host.txt; free -g >> $out/host.txt; nvidia-smi -L >> $out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 600 python bench.py --config C2 > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench c2 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "bench ref rc=$?" >> $out/rc.txt
