mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "same-key|within-3SE|safe|crop|passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | head -60
