# A/B pass: refill threshold (idle lane-iterations)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "same_key or crop" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('%.4e v/s  kernel %.1f ms frac %.3f ctr conn %d' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['counters']['conn_nonempty']))" 2>&1 | tail -1)"; }
for cfg in "5 256" "3 16"; do
  set -- $cfg
  BARGS="--config $1 --spp $2"
  for k in 4 8 16 32 64; do run c$1_w$k DTS_REFILL_K=$k; done
  run c$1_w16_nodefer DTS_REFILL_K=16 DTS_NO_DEFER=1
done
