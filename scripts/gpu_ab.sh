mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('%.4e v/s  kernel %.1f ms frac %.3f' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac']))" 2>&1 | tail -1)"; }
for cfg in "5 256" "3 16"; do
  set -- $cfg
  BARGS="--config $1 --spp $2"
  run c$1_b768
  run c$1_b896 DTS_LIB=libdts_b896.so
  run c$1_b1024 DTS_LIB=libdts_b1024.so
done
