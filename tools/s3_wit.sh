#!/bin/bash
# zero-row certificates: A/B probe + the partition parity tests
out=gpurun_out/${1:-s3wit}
mkdir -p $out
make -s -C paper_2605_05330_b200 > $out/build.log 2>&1
timeout 600 python tools/probe_witness.py --inst C5S18 --reps 1 > $out/w_c5s18.jsonl 2> $out/w_c5s18.err; echo "c5s18 rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C5S18 --reps 1 --exact > $out/w_c5s18x.jsonl 2> $out/w_c5s18x.err; echo "c5s18x rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C3 --reps 1 > $out/w_c3.jsonl 2> $out/w_c3.err; echo "c3 rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C2 --reps 1 > $out/w_c2.jsonl 2> $out/w_c2.err; echo "c2 rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/w_c5s24.jsonl 2> $out/w_c5s24.err; echo "c5s24 rc=$?" >> $out/rc.txt
timeout 900 python tools/probe_witness.py --inst C5S24 --reps 1 --dtype fp32 > $out/w_c5s24_32.jsonl 2> $out/w_c5s24_32.err; echo "c5s24 fp32 rc=$?" >> $out/rc.txt

cat $out/rc.txt
