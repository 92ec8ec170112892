#!/bin/bash
out=gpurun_out/${1:-s8}
mkdir -p $out
timeout 900 python -m pytest tests/test_witness_gpu.py tests/test_partition_gpu.py -m gpu -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/w_c5s24.jsonl 2> $out/w_c5s24.err; echo "probe rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_run.py --runs 2 > $out/run.jsonl 2> $out/run.err; echo "run rc=$?" >> $out/rc.txt
for it in 900 300; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s $it -c 1 -o $out/c5step_k$it python tools/probe_run.py > $out/ncu_k$it.log 2>&1; echo "ncu $it rc=$?" >> $out/rc.txt
done
cat $out/rc.txt; tail -3 $out/pytest.log; cut -c1-900 $out/w_c5s24.jsonl; cat $out/run.jsonl
