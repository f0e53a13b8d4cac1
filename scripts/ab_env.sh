# A/B of a launch-tuning environment variable: bash scripts/ab_env.sh VAR "v1 v2 ..." "configs"
VAR=$1; VALS=$2; CFGS=${3:-"5 3 4"}
for v in $VALS; do
 for c in $CFGS; do
  env $VAR=$v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$VAR=$v', $c, '%.4e' % d['value'], round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms'],3), flush=True)"
 done
done
