#!/bin/bash
# A/B of the partitioned step on C5 scale 24 (one part) under environment
# settings, one tools/probe_c5.py line per setting (the round-2 experiments in
# DESIGN.md section 4 were run this way):
#   tools/r02_ab.sh OUT "GN_PART_LONG=512" "GN_PART_CHUNK=0" "GN_LIB=exp/lib_h1.so" ...
# (A/B builds: make -C paper_2605_05330_b200 BUILD=build_x LIB=../exp/lib_x.so EXTRA=-D...)
out=gpurun_out/${1:-r2ab}
shift
mkdir -p $out
for env in "" "$@"; do
  env $env timeout 600 python tools/probe_c5.py --dtype ${DTYPE:-fp64} --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
