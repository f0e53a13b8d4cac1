# A/B of the deferred-connection kernels (queue size / CTA size builds) against the immediate default
run() { env "$@" timeout 300 python bench.py --config $C --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$* c$C', '%.4e' % d['value'], d['launch'], flush=True)"; }
for C in 5 3; do
 run DTS_LIB=libdts.so DTS_DEFER=0
 run DTS_LIB=libdts.so DTS_DEFER=1
 run DTS_LIB=libdts_d896q24.so DTS_DEFER=1
 run DTS_LIB=libdts_d832q28.so DTS_DEFER=1
 run DTS_LIB=libdts_d832q28.so DTS_DEFER=1 DTS_FLUSH_AT=20
 run DTS_LIB=libdts.so DTS_DEFER=0
done
