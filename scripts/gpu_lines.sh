# Bench lines of every config (through gpurun): configs 1-4 and 6 as the
# parity-case lines, config 5 (the default, with the MSE leg), and the
# paper-literal REUSE mode of configs 3 and 5.  Outputs gpurun_out/bench_TAG_*.json.
TAG=${1:-dev}
mkdir -p gpurun_out
for c in 1 2 3 4 6; do
  timeout 900 python bench.py --config $c --cpu-budget 10 > gpurun_out/bench_${TAG}_c$c.json 2> gpurun_out/bench_${TAG}_c$c.err; echo "bench c$c rc=$?"
done
for c in 3 5; do
  timeout 900 python bench.py --config $c --direction-mode reuse --no-cpu-baseline > gpurun_out/bench_${TAG}_c${c}_reuse.json 2> gpurun_out/bench_${TAG}_c${c}_reuse.err; echo "bench c$c reuse rc=$?"
done
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench c5 rc=$?"
