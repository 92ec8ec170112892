out=gpurun_out/s3v0
mkdir -p $out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?" >> $out/rc.txt
cat $out/rc.txt
