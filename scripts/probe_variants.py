"""Time the render kernel of each libdts_<variant>.so on configs 3 and 5 (reduced spp)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json, torch
sys.path.insert(0, ROOT)
import dts_inputs as I
from paper_2402_03106_b200 import dts
out = {}
for cfg, spp in ((3, 64), (5, 128)):
    c = I.as_f32(I.config(cfg)); c["spp"] = spp
    sc = dts.Scene(c); sc.table_build()
    h = torch.zeros(sc.hist_shape(), device="cuda"); ctr = torch.zeros(10, dtype=torch.int64, device="cuda")
    best = 1e30
    for it in range(3):
        h.zero_(); ctr.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); sc.render(spp, c["seed"] + it, 0, spp, h, None, ctr); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    v = int(ctr[2])
    out[cfg] = dict(ms=best, vps=v / best * 1e3, launch=dts.last_launch())
print(json.dumps(out))
'''.replace("ROOT", repr(ROOT))
variants = sys.argv[1:] or ["libdts.so"]
for v in variants:
    env = dict(os.environ, DTS_LIB=v)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
    print(v, r.stdout.strip() or r.stderr[-2000:], flush=True)
