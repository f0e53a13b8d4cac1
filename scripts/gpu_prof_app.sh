# ncu --set full of the connect-stage kernel (render_darts_kernel<..., RESUME>)
# in application replay mode (its kernel-replay metrics come back NaN), config 5
# on a 128 x 128 centre crop at spp 1024 (one chunk).
TAG=${1:-dev}
mkdir -p gpurun_out
PCMD="python bench.py --config 5 --spp 1024 --crop 128 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-mse"
$PCMD > gpurun_out/plain_app_${TAG}.log 2>&1 && \
  timeout 2400 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:render_darts \
    -s 3 -c 1 -o gpurun_out/prof_${TAG}_c5conn $PCMD > gpurun_out/ncu_app_${TAG}.log 2>&1; echo "ncu app rc=$?"
