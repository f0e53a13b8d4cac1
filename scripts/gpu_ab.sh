mkdir -p gpurun_out
DTS_LIB=libdts_checks.so timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import dts_inputs as I, torch
from paper_2402_03106_b200 import dts
for k in (3, 5):
    c = I.as_f32(I.config(k)); c = I.crop_center(c, 64, 64)
    sc = dts.Scene(c); sc.table_build()
    h, _, ctr = dts.render_to_tensor(sc, c['spp'], 1); torch.cuda.synchronize()
    print(k, dts.counters_dict(ctr), 'check failures', dts.check_failures())
" > gpurun_out/checks_full.log 2>&1; echo "checks rc=$?"; cat gpurun_out/checks_full.log | tail -3
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
run() { tag=$1; shift; env "$@" timeout 600 $B $BARGS > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('%.4e v/s  kernel %.1f ms frac %.3f' % (d['value'], d['roofline']['kernel_ms'], d['roofline']['frac']))" 2>&1 | tail -1)"; }
for cfg in "5 256" "3 16"; do
  set -- $cfg
  BARGS="--config $1 --spp $2"
  run c$1_def
  run c$1_f24 DTS_FLUSH_AT=24
  run c$1_nodefer DTS_NO_DEFER=1
done
