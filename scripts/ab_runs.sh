# A/B of bench runs given as "label|ENV=val ...|configs[|extra bench args]" specs,
# two alternating rounds:
#   bash scripts/ab_runs.sh TAG "one|DTS_WAVEFRONT=0|5 3" "two|DTS_WAVEFRONT=1|5 3|--spp 128"
TAG=$1; shift
mkdir -p gpurun_out
for round in 1 2; do
  for spec in "$@"; do
    IFS='|' read -r label envs cfgs extra <<< "$spec"
    for c in $cfgs; do
      env $envs timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e $extra 2>gpurun_out/ab_${TAG}_${label}_c${c}_r${round}.err | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['counters']; print('$label', 'cfg$c', 'round$round', '%.4e' % d['value'], 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.2f' % d['roofline']['kernel_ms'], 'ms/step %.2f' % d['ms_per_step'], 'paths', k['paths'], 'verts', k['vertices'], 'walk %.4f' % (k.get('walk_vertices', 0) / max(k['vertices'], 1)), 'launches', d['launch'], 'sm', d['clocks']['sm_mhz'], d['clocks']['reasons'])" || echo "$label cfg$c FAILED"
    done
  done
done | tee gpurun_out/ab_${TAG}.log
