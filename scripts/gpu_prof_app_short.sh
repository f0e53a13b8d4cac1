# ncu --set full of the connect-stage kernel of a short-walk REUSE config
# (CFG, default 4) in application replay mode (kernel replay returns NaN for
# the hand-off consumers); one capture per gpurun call (64 MiB copy-back limit)
TAG=${1:-dev}
C=${CFG:-4}
mkdir -p gpurun_out
PCMD="python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-mse"
$PCMD > gpurun_out/plain_app_c${C}_${TAG}.log 2>&1 && \
  timeout 2400 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:render_darts \
    -s 3 -c 1 -o gpurun_out/prof_${TAG}_c${C}conn $PCMD > gpurun_out/ncu_app_c${C}_${TAG}.log 2>&1; echo "ncu app rc=$?"
