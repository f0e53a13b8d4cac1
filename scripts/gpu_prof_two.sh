# ncu --set full of the two kernels of one chunk of a two-stage render (start or
# walk stage + connect stage) for config CFG (default 4); one capture per call
#   CFG=4 bash scripts/gpu_prof_two.sh TAG
TAG=${1:-dev}
C=${CFG:-4}
mkdir -p gpurun_out
PCMD="python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-mse ${EXTRA:-}"
$PCMD > gpurun_out/plain_two_c${C}_${TAG}.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"render_darts|start_kernel|walk_kernel" -s 6 -c 2 \
    -o gpurun_out/prof_${TAG}_c$C $PCMD > gpurun_out/ncu_two_c${C}_${TAG}.log 2>&1; echo "ncu c$C rc=$?"
