mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_p2p.py -m gpu -q -x -s > gpurun_out/pytest_p2p.log 2>&1; echo "p2p rc=$?"; tail -15 gpurun_out/pytest_p2p.log
timeout 600 python bench.py --steps 1 --warmup 3 --spp 64 --no-cpu-baseline > gpurun_out/b.json 2>&1; echo "bench rc=$?"; tail -c 300 gpurun_out/b.json
