mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
DTS_LIB=libdts_risB.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "same_key or crop or sharding" > gpurun_out/pytest_risB.log 2>&1; echo "pytest risB rc=$?"
grep -E "same-key|crop|passed|failed" gpurun_out/pytest_risB.log | head -20
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('%.4e v/s  kernel %.1f ms frac %.3f ctr conn %d' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['counters']['conn_nonempty']))" 2>&1 | tail -1)"; }
for cfg in "5 256" "3 16" "4 256" "2 16"; do
  set -- $cfg
  BARGS="--config $1 --spp $2"
  run c$1_A
  run c$1_B DTS_LIB=libdts_risB.so
  run c$1_B640 DTS_LIB=libdts_risB640.so
done
