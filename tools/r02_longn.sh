#!/bin/bash
# long-row threshold vs part size: C3 (2M entries, one part), C5 8-way parts (65M), C5 one part (520M)
out=gpurun_out/${1:-r2longn}
mkdir -p $out
for L in 32 64 128 256 512 1024; do
  GN_PART_LONG=$L timeout 600 python tools/probe_engines.py --config C3 >> $out/c3.jsonl 2>> $out/c3.err
done
for L in 128 256 512 1024; do
  GN_PART_LONG=$L timeout 900 python tools/probe_scaling.py --gpus 8 --parts 0,3,7 --iters 30 > $out/n8_L$L.json 2>> $out/n8.err
done
