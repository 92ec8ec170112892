#!/bin/bash
# Round-2 GPU test pass: the new full-budget and drop-in tests first (timed), then the whole -m gpu suite.
out=gpurun_out/${1:-r2t}
mkdir -p $out
export GN_EXCURSION_DIR=$out/fp32_excursions
timeout 1800 python -m pytest tests/test_dropin_reference_gpu.py tests/test_fullbudget_gpu.py tests/test_partition_gpu.py -q --durations=0 -x > $out/new_tests.log 2>&1; echo "new rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $out/pytest.log 2>&1; echo "all rc=$?" >> $out/rc.txt
