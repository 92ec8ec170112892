#!/bin/bash
# Round-2 measurement pass: C5 step probes (fp64/fp32), the direct halo on one
# GPU (3 parts, store sectors per pushed value), one ncu --set full capture of
# the C5 step kernel, the other configs' bench lines and the default bench's
# launch list.  Outputs under gpurun_out/$1.
out=gpurun_out/${1:-r2m}
mkdir -p $out
for dt in fp64 fp32; do timeout 600 python tools/probe_c5.py --dtype $dt >> $out/probe.jsonl 2>> $out/probe.err; done
timeout 600 python tools/probe_halo.py --scale 22 --parts 3 > $out/halo.json 2> $out/halo.err
timeout 900 ncu --nvtx --nvtx-include "push_probe/" --metrics \
  l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,gpu__time_duration.sum \
  --csv --log-file $out/halo_ncu.csv python tools/probe_halo.py --scale 22 --parts 3 > $out/halo_ncu.log 2>&1
echo "halo ncu rc=$?" >> $out/rc.txt
for c in C3 C4; do timeout 900 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c rc=$?" >> $out/rc.txt; done
timeout 900 python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_part_step" -s 0 -c 1 \
    -o $out/c5step python tools/probe_c5.py --dtype fp64 --reps 1 --iters 20 > $out/ncu.log 2>&1
echo "ncu step rc=$?" >> $out/rc.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/launches.log 2>&1
echo "launches rc=$?" >> $out/rc.txt
