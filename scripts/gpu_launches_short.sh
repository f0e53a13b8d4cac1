# ncu launch lists (time per launch) of short-walk configs' bench commands
# (CFGS, default "4 2"): the split of a step between the start and connect stages
TAG=${1:-dev}
mkdir -p gpurun_out
for c in ${CFGS:-4 2}; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-mse"
  $CMD > gpurun_out/plain_launch_c${c}_${TAG}.log 2>&1 && \
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/launches_c${c}_${TAG}.csv $CMD > gpurun_out/ncu_launch_c${c}_${TAG}.log 2>&1; echo "ncu-launch c$c rc=$?"
done
