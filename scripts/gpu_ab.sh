B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));c=d['counters'];print('%.4e v/s  kernel %.1f ms frac %.3f block %d' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['launch']['block']))" 2>&1 | tail -1)"; }
BARGS="--config 5 --spp 256"
run c5_d1 DTS_DEFER=1
run c5_d0 DTS_DEFER=0
run c5_d1b DTS_DEFER=1
run c5_d0b DTS_DEFER=0
BARGS="--config 3 --spp 16"
run c3_d1 DTS_DEFER=1
run c3_d0 DTS_DEFER=0
