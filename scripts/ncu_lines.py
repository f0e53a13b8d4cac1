#!/usr/bin/env python
"""Per-source-region instruction accounting of an ncu --set full capture
(`ncu -i REP --page source --csv --print-source cuda,sass`): warp-instructions
per vertex and SIMT efficiency by source line / region of darts_vertex.

    python scripts/ncu_lines.py REP VERTICES [kernel=REGEX] [name:file:lo:hi ...]"""
import collections
import csv
import subprocess
import sys

rep, verts = sys.argv[1], float(sys.argv[2])
kern = []
if len(sys.argv) > 3 and sys.argv[3].startswith("kernel="):   # e.g. kernel=walk_kernel (a regex)
    kern = ["-k", "regex:" + sys.argv[3].split("=", 1)[1]]
    del sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", *kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
agg, thr, st, src = collections.Counter(), collections.Counter(), collections.Counter(), {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 10 or r[0] in ("Line No", "Function Name"):
        continue
    try:
        ln, e, t, w = int(r[0]), int(r[7]), int(r[8]), int(r[4])
    except ValueError:
        continue
    agg[(cur, ln)] += e
    thr[(cur, ln)] += t
    st[(cur, ln)] += w
    src[(cur, ln)] = r[1][:100]
tot = sum(agg.values())
print(f"total warp-inst/vertex {tot / verts:.2f}  thread-inst/vertex {sum(thr.values()) / verts:.1f}")
if len(sys.argv) > 3:
    for spec in sys.argv[3:]:
        name, f, a, b = spec.split(":")
        a, b = int(a), int(b)
        e = sum(v for (ff, l), v in agg.items() if ff == f and a <= l <= b)
        t = sum(v for (ff, l), v in thr.items() if ff == f and a <= l <= b)
        print(f"{name:24s} {e / verts:6.2f} warp/vtx  simt {t / max(e, 1):5.1f}")
print()
for k, e in agg.most_common(int(__import__("os").environ.get("NCU_LINES_TOP", "40"))):
    print(f"{k[0]:16s} {k[1]:5d} {e / verts:6.3f} simt {thr[k] / e:5.1f}  {src[k]}")
