# Full GPU pass of a round (run through gpurun): memory-safety check build,
# pytest -m gpu, smoke, bench lines of every config, the ncu launch list (+ DRAM
# bytes) of the default bench command, ncu --set full of the render kernel.
# Outputs land in gpurun_out/; copy what is to be kept into profiles/.
set -x
TAG=${1:-dev}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_info.txt
bash scripts/build_variants.sh "checks:-DDTS_CHECKS=1" > /dev/null 2>&1
DTS_LIB=libdts_checks.so timeout 300 python scripts/sanitize_case.py > gpurun_out/checks.log 2>&1; echo "checks rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in 1 2 3 4 6; do
  timeout 900 python bench.py --config $c --cpu-budget 10 > gpurun_out/bench_${TAG}_c$c.json 2> gpurun_out/bench_${TAG}_c$c.err
done
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench rc=$?"
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_c5_${TAG}.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
bash scripts/gpu_prof.sh $TAG
