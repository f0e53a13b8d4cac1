mkdir -p gpurun_out
timeout 1800 python scripts/sweeps.py > gpurun_out/sweeps.log 2>&1; echo "sweeps rc=$?"; cat gpurun_out/sweeps.log | tail -14
timeout 1200 python scripts/response_experiment.py > gpurun_out/response.log 2>&1; echo "resp rc=$?"; cat gpurun_out/response.log | tail -4
