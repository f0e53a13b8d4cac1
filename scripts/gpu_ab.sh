mkdir -p gpurun_out
DTS_LIB=libdts_checks.so timeout 300 python scripts/sanitize_case.py > gpurun_out/checks.log 2>&1; echo "checks rc=$?"; tail -1 gpurun_out/checks.log
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));c=d['counters'];print('%.4e v/s  kernel %.1f ms frac %.3f block %d' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['launch']['block']))" 2>&1 | tail -1)"; }
for cfg in "5 256" "3 16" "4 256" "2 16"; do
  set -- $cfg
  BARGS="--config $1 --spp $2"
  run c$1_v53
done
