#!/bin/bash
out=gpurun_out/${1:-s7}
mkdir -p $out
timeout 1200 python -m pytest tests/test_witness_gpu.py tests/test_partition_gpu.py tests/test_ipc_gpu.py tests/test_fuzz_gpu.py -m gpu -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/w_c5s24.jsonl 2> $out/w_c5s24.err; echo "probe rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_active.py > $out/active.json 2> $out/active.err; echo "active rc=$?" >> $out/rc.txt
cat $out/rc.txt; tail -6 $out/pytest.log; cut -c1-900 $out/w_c5s24.jsonl; cat $out/active.json
