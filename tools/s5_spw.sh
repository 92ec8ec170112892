#!/bin/bash
# slices per warp (GN_PART_SPW) A/B on C5 scale 24, after the certificate tests
out=gpurun_out/${1:-s5}
mkdir -p $out
timeout 1200 python -m pytest tests/test_witness_gpu.py tests/test_partition_gpu.py -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
for spw in 1 4 16 64; do
  GN_PART_SPW=$spw timeout 900 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/w_c5s24_spw$spw.jsonl 2> $out/w_c5s24_spw$spw.err; echo "spw $spw rc=$?" >> $out/rc.txt
done
cat $out/rc.txt; tail -5 $out/pytest.log
for spw in 1 4 16 64; do echo "== spw $spw"; cut -c1-700 $out/w_c5s24_spw$spw.jsonl; done
