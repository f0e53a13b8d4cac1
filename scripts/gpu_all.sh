# every config's bench line, equal-time MSE harness, full-launch DRAM traffic of the render kernel
mkdir -p gpurun_out
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --cpu-budget 10 > gpurun_out/bench_all_c$c.json 2> gpurun_out/bench_all_c$c.err; echo "bench c$c rc=$?"
done
timeout 1800 python scripts/mse_equal_time.py --reps 4 > gpurun_out/mse.log 2>&1; echo "mse rc=$?"; cat gpurun_out/mse.log | tail -8
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_traffic.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:render_darts -s 3 -c 1 --csv --log-file gpurun_out/traffic_c5.csv $CMD > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
