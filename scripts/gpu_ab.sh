mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -s -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "response|passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | cut -c1-250 | head -20
timeout 1200 python scripts/response_experiment.py > gpurun_out/response.log 2>&1; echo "resp rc=$?"; cat gpurun_out/response.log | tail -4
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $B --config 5 --spp 256 > gpurun_out/ab_c5.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/ab_c5.json'));print('c5 %.4e' % d['value'])"
