mkdir -p gpurun_out
DTS_LIB=libdts_checks.so timeout 300 python scripts/sanitize_case.py > gpurun_out/checks.log 2>&1; echo "checks rc=$?"; tail -3 gpurun_out/checks.log
DTS_LIB=libdts_checks.so timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import dts_inputs as I, torch
from paper_2402_03106_b200 import dts
for k in (3, 5):
    c = I.as_f32(I.config(k)); c = I.crop_center(c, 64, 64)
    sc = dts.Scene(c); sc.table_build()
    h, _, ctr = dts.render_to_tensor(sc, c['spp'], 1); torch.cuda.synchronize()
    print(k, dts.counters_dict(ctr)['vertices'], 'check failures', dts.check_failures())
" > gpurun_out/checks_full.log 2>&1; echo "checks full rc=$?"; cat gpurun_out/checks_full.log | tail -3
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
