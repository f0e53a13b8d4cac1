# Fraction of medium vertices whose connection provably cannot land in the bin
# (diagnostic build libdts_skipcount.so: counters 'rejected' = cheap bound,
# 'nonfinite' = box-corner bound)
for c in 5 3; do
  DTS_LIB=libdts_skipcount.so timeout 600 python bench.py --config $c --steps 1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['counters']; print('cfg$c', 'vertices', k['vertices'], 'skip_cheap %.4f' % (k['rejected']/k['vertices']), 'skip_corner %.4f' % (k['nonfinite']/k['vertices']))"
done | tee gpurun_out/skipcount.log
