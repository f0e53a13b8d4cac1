# A/B of library variants on the bench (through gpurun): scripts/ab_libs.sh TAG CONFIGS LIB...
# e.g. scripts/ab_libs.sh x2 "5 3" libdts.so libdts_scalar.so   (two alternating rounds)
TAG=$1; CFGS=$2; shift 2
mkdir -p gpurun_out
for round in 1 2; do
  for lib in "$@"; do
    for c in $CFGS; do
      DTS_LIB=$lib timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'cfg$c', 'round$round', '%.4e' % d['value'], 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.2f' % d['roofline']['kernel_ms'], 'sm_mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done | tee gpurun_out/ab_${TAG}.log
