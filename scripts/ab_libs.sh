# A/B of in-tree library builds: bash scripts/ab_libs.sh libdts.so libdts_<variant>.so ... (bench configs 5, 3, 4)
for lib in "$@"; do
 for c in 5 3 4; do
  DTS_LIB=$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', $c, d['value'], round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], flush=True)"
 done
done
