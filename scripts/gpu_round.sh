# full GPU pass: tests, bench lines, ncu launch list and one full capture of the render kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_info.txt
lscpu | head -20 > gpurun_out/cpu_info.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -s -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench5 rc=$?"
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench3 rc=$?"
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
PCMD="python bench.py --config 5 --spp 16 --steps 1 --warmup 3 --no-cpu-baseline"
$PCMD > gpurun_out/plain_prof.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_darts -s 3 -c 1 -o gpurun_out/prof_c5_render $PCMD > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
