mkdir -p gpurun_out/v1
nvidia-smi > gpurun_out/v1/smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/v1/pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1/smoke.log 2>&1; echo "smoke rc=$?"
