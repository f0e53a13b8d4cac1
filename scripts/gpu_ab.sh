mkdir -p gpurun_out
DTS_LIB=libdts_checks.so timeout 300 python scripts/sanitize_case.py > gpurun_out/checks.log 2>&1; echo "checks rc=$?"; tail -1 gpurun_out/checks.log
DTS_LIB=libdts_checks.so DTS_DEFER=1 timeout 300 python scripts/sanitize_case.py > gpurun_out/checks_defer.log 2>&1; echo "checks defer rc=$?"; tail -1 gpurun_out/checks_defer.log
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
DTS_DEFER=1 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "same_key or crop or sharding or host" > gpurun_out/pytest_gpu_defer.log 2>&1; echo "pytest defer rc=$?"; tail -1 gpurun_out/pytest_gpu_defer.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --cpu-budget 10 > gpurun_out/bench_v5_c$c.json 2> gpurun_out/bench_v5_c$c.err; echo "bench c$c rc=$?"; done
timeout 900 python bench.py > gpurun_out/bench_v5_c5.json 2> gpurun_out/bench_v5_c5.err; echo "bench c5 rc=$?"
for c in 1 2 3 4 5; do python -c "
import json; d=json.load(open('gpurun_out/bench_v5_c$c.json')); print($c, '%.4e'%d['value'], '%.2f ms'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.3e'%d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['launch']['smem'])"; done
