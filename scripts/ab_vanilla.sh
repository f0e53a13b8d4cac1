# vanilla kernel: per-warp shared-memory rows (default) against direct REDs
for round in 1 2; do
  for rows in 1 0; do
    for spec in "4 256" "3 64" "5 16" "1 4096"; do
      set -- $spec
      DTS_VANILLA_ROWS=$rows timeout 600 python bench.py --config $1 --strategy vanilla --spp $2 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rows=$rows', 'cfg$1 spp$2 round$round', 'paths/s %.4e' % d['paths_per_s'], 'vertices/s %.4e' % d['value'], 'ms/step %.2f' % d['ms_per_step'])"
    done
  done
done | tee gpurun_out/ab_vanilla.log
