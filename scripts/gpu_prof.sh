# ncu --set full captures of the render kernel, config 5 at spp 16 and config 3 at spp 4 (tag = $1)
TAG=${1:-dev}
mkdir -p gpurun_out
for spec in "5 16" "3 4"; do
  set -- $spec
  PCMD="python bench.py --config $1 --spp $2 --steps 1 --warmup 3 --no-cpu-baseline"
  $PCMD > gpurun_out/plain_prof_c$1.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_darts -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_c$1 $PCMD > gpurun_out/ncu_full_c$1.log 2>&1; echo "ncu c$1 rc=$?"
done
