mkdir -p gpurun_out
timeout 1800 python scripts/mse_vs_oracle.py > gpurun_out/mse_vs_oracle.log 2>&1; echo "rc=$?"; cat gpurun_out/mse_vs_oracle.log | tail -8
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "debug_parity" > gpurun_out/pytest_dbg.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_dbg.log
