# Bench lines of every config (through gpurun): configs 1-4 and 6 as the
# parity-case lines (enough steps for >= 1 s of timed region, so that the
# nvidia-smi clock sampler sees the run), config 5 (the default, with the MSE
# leg), and the paper-literal REUSE mode of configs 3 and 5.
TAG=${1:-dev}
mkdir -p gpurun_out
for spec in "1 2000" "2 500" "3 3" "4 100" "6 500"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --steps $2 --cpu-budget 10 > gpurun_out/bench_${TAG}_c$1.json 2> gpurun_out/bench_${TAG}_c$1.err; echo "bench c$1 rc=$?"
done
for c in 3 5; do
  timeout 900 python bench.py --config $c --direction-mode reuse --no-cpu-baseline > gpurun_out/bench_${TAG}_c${c}_reuse.json 2> gpurun_out/bench_${TAG}_c${c}_reuse.err; echo "bench c$c reuse rc=$?"
done
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench c5 rc=$?"
