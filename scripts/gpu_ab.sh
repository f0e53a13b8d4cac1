mkdir -p gpurun_out
DTS_LIB=libdts_checks.so timeout 300 python scripts/sanitize_case.py > gpurun_out/checks.log 2>&1; echo "checks rc=$?"; tail -1 gpurun_out/checks.log
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --cpu-budget 10 > gpurun_out/bench_v6_c$c.json 2> gpurun_out/bench_v6_c$c.err; echo "bench c$c rc=$?"; done
timeout 900 python bench.py > gpurun_out/bench_v6_c5.json 2> gpurun_out/bench_v6_c5.err; echo "bench c5 rc=$?"
for c in 1 2 3 4 5; do python -c "
import json; d=json.load(open('gpurun_out/bench_v6_c$c.json')); print($c, '%.4e'%d['value'], '%.2f ms'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.3e'%d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['launch'])"; done
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5_v6.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
bash scripts/gpu_prof.sh v6 > /dev/null 2>&1; echo "prof rc=$?"
