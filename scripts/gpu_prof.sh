# ncu evidence of a round (run through gpurun, one GPU): with LAUNCH=1 the launch
# list of the default bench command (per-launch time + DRAM bytes), then
# `ncu --set full` of the render kernels for each "config spp" spec (one chunk of
# the two-stage render: the walk kernel and the connect kernel).  Keep one
# capture per gpurun call: the copy-back limit is 64 MiB.
#   bash scripts/gpu_prof.sh TAG "5 128" ["3 4" ...]
TAG=${1:-dev}; shift
mkdir -p gpurun_out
if [ "${LAUNCH:-0}" = "1" ]; then
  CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-mse"
  $CMD > gpurun_out/plain_launch_${TAG}.log 2>&1 && \
    timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/launches_c5_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "ncu-launch rc=$?"
fi
for spec in "$@"; do
  set -- $spec
  PCMD="python bench.py --config $1 --spp $2 ${CROP:+--crop $CROP} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-mse"
  $PCMD > gpurun_out/plain_prof_c$1_${TAG}.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"walk_kernel|render_darts" -s 6 -c 2 \
      -o gpurun_out/prof_${TAG}_c$1 $PCMD > gpurun_out/ncu_full_c$1_${TAG}.log 2>&1; echo "ncu c$1 rc=$?"
done
