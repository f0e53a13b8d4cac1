mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -s -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | head -20
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('%.4e v/s  kernel %.1f ms frac %.3f ctr conn %d' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['counters']['conn_nonempty']))" 2>&1 | tail -1)"; }
for cfg in "5 256" "3 16"; do
  set -- $cfg
  BARGS="--config $1 --spp $2"
  run c$1_def
  run c$1_nodefer DTS_NO_DEFER=1
  run c$1_b640 DTS_LIB=libdts_b640.so
done
