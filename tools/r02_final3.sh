#!/bin/bash
# Round-2 closing pass on the final step kernel: the -m gpu suite, the C5 bench
# lines (fp64 default, fp32), the certificate A/B in both precisions, ncu of the
# step at three stages and of the plain kernel, the metrics sweep of one
# pursuit, the default bench's launch list, the plain-kernel scaling projection.
out=gpurun_out/${1:-r2f3}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --dtype fp32 --no-cpu-baseline > $out/bench_c5_fp32.json 2> $out/bench_c5_fp32.err; echo "bench c5 fp32 rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/witness_ab.jsonl 2> $out/witness_ab.err; echo "witness ab rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C5S24 --reps 1 --dtype fp32 > $out/witness_ab_fp32.jsonl 2> $out/witness_ab_fp32.err; echo "witness ab fp32 rc=$?" >> $out/rc.txt
for it in 5 300 900; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s $it -c 1 -o $out/c5step_k$it python tools/probe_run.py > $out/ncu_k$it.log 2>&1; echo "ncu $it rc=$?" >> $out/rc.txt
done
GN_PART_WITNESS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s 5 -c 1 -o $out/c5step_plain python tools/probe_run.py --iters 20 > $out/ncu_plain.log 2>&1; echo "ncu plain rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_part" --csv --log-file $out/sweep.csv python tools/probe_run.py > $out/sweep.log 2>&1; echo "sweep rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-certificate-report > $out/launches.log 2>&1; echo "launches rc=$?" >> $out/rc.txt
GN_PART_WITNESS=0 timeout 1200 python tools/probe_scaling.py --scale 24 --iters 30 > $out/scaling.json 2> $out/scaling.err; echo "scaling rc=$?" >> $out/rc.txt
cat $out/rc.txt
