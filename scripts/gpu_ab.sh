mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -s -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "same-key|cfg.*safe|passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | cut -c1-200 | head -40
timeout 2400 python scripts/mse_equal_time.py --reps 4 > gpurun_out/mse.log 2>&1; echo "mse rc=$?"; cat gpurun_out/mse.log | tail -8
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $B --config 5 --spp 256 > gpurun_out/ab_c5.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/ab_c5.json'));print('c5 %.4e' % d['value'])"
