#!/bin/bash
# The long-row chunk length A/B (GN_PART_CHUNK, default 128 -> 512) as a full
# pass before the default moves: the -m gpu suite, the C5 bench lines, the
# plain kernel's ncu capture, the metrics sweep of one pursuit and the launch
# list, all under the environment setting.
out=gpurun_out/${1:-r2f6}
mkdir -p $out
export GN_PART_CHUNK=${CHUNK:-512}
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 1800 python -m pytest tests -m gpu -q --durations=5 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --dtype fp32 --no-cpu-baseline > $out/bench_c5_fp32.json 2> $out/bench_c5_fp32.err; echo "bench c5 fp32 rc=$?" >> $out/rc.txt
GN_PART_WITNESS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s 5 -c 1 -o $out/c5step_plain python tools/probe_run.py --iters 20 > $out/ncu_plain.log 2>&1; echo "ncu plain rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_part" --csv --log-file $out/sweep.csv python tools/probe_run.py > $out/sweep.log 2>&1; echo "sweep rc=$?" >> $out/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-certificate-report > $out/launches.log 2>&1; echo "launches rc=$?" >> $out/rc.txt
cat $out/rc.txt
