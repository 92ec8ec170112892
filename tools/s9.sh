#!/bin/bash
out=gpurun_out/${1:-s9}
mkdir -p $out
timeout 900 python -m pytest tests/test_witness_gpu.py tests/test_partition_gpu.py -m gpu -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/w_c5s24.jsonl 2> $out/w_c5s24.err; echo "probe rc=$?" >> $out/rc.txt
cat $out/rc.txt; tail -3 $out/pytest.log; cut -c1-900 $out/w_c5s24.jsonl
