# Quick GPU pass (run through gpurun): pytest -m gpu with the tests' printed
# parity figures, smoke, and one default bench line.  Outputs in gpurun_out/.
TAG=${1:-dev}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_info.txt
DTS_DUMP_DIR=gpurun_out/dump_${TAG} timeout 2400 python -m pytest tests -m gpu -q -s -rf > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 3 > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench rc=$?"
fi
