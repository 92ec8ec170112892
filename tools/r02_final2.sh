#!/bin/bash
# Round-2 final measurement pass (after the certificates / settled rows):
# smoke, the -m gpu suite, every bench line, the reference arm, the default
# bench's launch list, ncu --set full of the C5 step at three stages of the
# pursuit and with the certificates off, and a metrics sweep over every launch
# of one pursuit (sectors and DRAM bytes per iteration).
out=gpurun_out/${1:-r2f2}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
nproc > $out/host.txt; nvidia-smi -L >> $out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --dtype fp32 --no-cpu-baseline > $out/bench_c5_fp32.json 2> $out/bench_c5_fp32.err; echo "bench c5 fp32 rc=$?" >> $out/rc.txt
for c in C2 C3 C4; do timeout 900 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c rc=$?" >> $out/rc.txt; done
timeout 900 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "bench ref rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_witness.py --inst C5S24 --reps 1 > $out/witness_ab.jsonl 2> $out/witness_ab.err; echo "witness ab rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_active.py > $out/active.json 2> $out/active.err; echo "active rc=$?" >> $out/rc.txt
timeout 600 python tools/probe_run.py --runs 2 > $out/run.jsonl 2> $out/run.err; echo "run rc=$?" >> $out/rc.txt
for it in 5 300 900; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s $it -c 1 -o $out/c5step_k$it python tools/probe_run.py > $out/ncu_k$it.log 2>&1; echo "ncu $it rc=$?" >> $out/rc.txt
done
GN_PART_WITNESS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s 5 -c 1 -o $out/c5step_plain python tools/probe_run.py --iters 20 > $out/ncu_plain.log 2>&1; echo "ncu plain rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_part" --csv --log-file $out/sweep.csv python tools/probe_run.py > $out/sweep.log 2>&1; echo "sweep rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-certificate-report > $out/launches.log 2>&1; echo "launches rc=$?" >> $out/rc.txt
cat $out/rc.txt
