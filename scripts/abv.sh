# A/B timing of prebuilt library variants (no build, no tests): VARIANTS="v0 v1" CONFIGS="2 4" REPS=2
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-1}); do
for c in ${CONFIGS:-2}; do
  for v in ${VARIANTS}; do
    lib=paper_2101_11408_b200/libfpparse_$v.so; [ "$v" = product ] && lib=""
    FPP_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS} > gpurun_out/abv_${v}_c$c.json 2>gpurun_out/abv_${v}_c$c.err
    python - <<PY
import json
try:
    d=json.loads(open('gpurun_out/abv_${v}_c$c.json').read().strip().splitlines()[-1])
    print('%-10s c$c'%'$v', 'ms %.3f'%d['ms_per_step'], 'kern %.3f'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'], 'mism', d['parity']['mismatches'], 'mhz', d['clocks']['sm_mhz'])
except Exception as e:
    print('$v c$c failed', e)
PY
  done
done
done
