# ncu --set full of the one-stage render kernel on a short-walk config (CFGS, default 4;
# one capture per gpurun call: the copy-back limit is 64 MiB)
TAG=${1:-dev}
mkdir -p gpurun_out
for c in ${CFGS:-4}; do
  PCMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-mse"
  $PCMD > gpurun_out/plain_short_c${c}_${TAG}.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_darts -s 3 -c 1 \
      -o gpurun_out/prof_${TAG}_c$c $PCMD > gpurun_out/ncu_short_c${c}_${TAG}.log 2>&1; echo "ncu c$c rc=$?"
done
