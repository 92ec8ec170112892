#!/bin/bash
# After a change to the small kernels of the partitioned iteration (combine,
# witness, settle): the -m gpu suite, the C5 bench lines, the certificate A/B,
# the metrics sweep of one pursuit and the default bench's launch list (the
# step kernel's own ncu captures stay valid).
out=gpurun_out/${1:-r2f4}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --dtype fp32 --no-cpu-baseline > $out/bench_c5_fp32.json 2> $out/bench_c5_fp32.err; echo "bench c5 fp32 rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/witness_ab.jsonl 2> $out/witness_ab.err; echo "witness ab rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_part" --csv --log-file $out/sweep.csv python tools/probe_run.py > $out/sweep.log 2>&1; echo "sweep rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-certificate-report > $out/launches.log 2>&1; echo "launches rc=$?" >> $out/rc.txt
cat $out/rc.txt
