mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "same_key or crop" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
DTS_LIB=libdts_inner2.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "same_key or crop" > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest inner2 rc=$?"; tail -1 gpurun_out/pytest_gpu2.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('%.4e v/s  kernel %.1f ms frac %.3f' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac']))" 2>&1 | tail -1)"; }
for cfg in "5 256" "3 16" "4 256"; do
  set -- $cfg
  BARGS="--config $1 --spp $2"
  run c$1_i1
  run c$1_i2 DTS_LIB=libdts_inner2.so
  run c$1_i2_f24 DTS_LIB=libdts_inner2.so DTS_FLUSH_AT=24
  run c$1_i3_f20 DTS_LIB=libdts_inner3.so DTS_FLUSH_AT=20
done
