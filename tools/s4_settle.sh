#!/bin/bash
# settled rows: the certificate/settle tests, the partition suites, the A/B probe
out=gpurun_out/${1:-s4}
mkdir -p $out
timeout 1200 python -m pytest tests/test_witness_gpu.py tests/test_partition_gpu.py tests/test_ipc_gpu.py -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C5S18 --reps 1 > $out/w_c5s18.jsonl 2> $out/w_c5s18.err; echo "c5s18 rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/w_c5s24.jsonl 2> $out/w_c5s24.err; echo "c5s24 rc=$?" >> $out/rc.txt
timeout 900 python -m pytest tests/test_fullbudget_gpu.py -m gpu -x -q -k "C5 or c5" > $out/pytest_full.log 2>&1; echo "pytest full rc=$?" >> $out/rc.txt
cat $out/rc.txt; tail -15 $out/pytest.log; cat $out/w_c5s24.jsonl; tail -3 $out/pytest_full.log
