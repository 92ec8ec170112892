#!/bin/bash
# chunk/threshold sweep; partition tests; scaling projection (balanced ranges, hubs-first ghosts)
out=gpurun_out/${1:-r2chunk}
mkdir -p $out
timeout 1200 python -m pytest tests/test_partition_gpu.py tests/test_ipc_gpu.py -q -x > $out/part_tests.log 2>&1; echo "part tests rc=$?" >> $out/rc.txt
for env in "GN_PART_CHUNK=0" "GN_PART_CHUNK=128" "GN_PART_CHUNK=64 GN_PART_LONG=2048" "GN_PART_CHUNK=128 GN_PART_LONG=2048" "GN_PART_CHUNK=128 GN_PART_LONG=1024" "GN_PART_CHUNK=256 GN_PART_LONG=1024"; do
  env $env timeout 600 python tools/probe_c5.py --dtype fp64 --reps 5 >> $out/probe.jsonl 2>> $out/probe.err
done
timeout 1200 python tools/probe_scaling.py --scale 24 --iters 30 --gpus 1,2,8 > $out/scaling.json 2> $out/scaling.err; echo "scaling rc=$?" >> $out/rc.txt
GN_PART_CHUNK=128 GN_PART_LONG=2048 timeout 1200 python tools/probe_scaling.py --scale 24 --iters 30 --gpus 1,8 > $out/scaling_chunk.json 2> $out/scaling_chunk.err; echo "scaling chunk rc=$?" >> $out/rc.txt
