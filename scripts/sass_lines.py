"""Static SASS instruction counts per source line of one kernel (nvdisasm -g
output, see scripts/sass_of.sh): python scripts/sass_lines.py k.sass [file lo hi]."""
import collections
import re
import sys

lines = open(sys.argv[1]).read().split("\n")
cur = None
cnt = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for ln in lines:
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", ln)
    if m and cur:
        cnt[cur] += 1
        ops[cur][m.group(2) + (m.group(3) or "")] += 1
print("total", sum(cnt.values()))
if len(sys.argv) > 4:
    f, lo, hi = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    sel = sorted((k, v) for k, v in cnt.items() if k[0] == f and lo <= k[1] <= hi)
    print("region", sum(v for _, v in sel))
    agg = collections.Counter()
    for k, v in sel:
        agg.update(ops[k])
        print(k[1], v, dict(ops[k]))
    print("ops", dict(agg.most_common()))
