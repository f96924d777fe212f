# A/B of prebuilt variants on config 5/7 with per-kernel times from the bench line: VARIANTS="product sa1"
mkdir -p gpurun_out
for c in ${CONFIGS:-5 7}; do
  for v in ${VARIANTS}; do
    lib=paper_2101_11408_b200/libfpparse_$v.so; [ "$v" = product ] && lib=""
    FPP_LIB=$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abv_${v}_c$c.json 2>gpurun_out/abv_${v}_c$c.err
    python - <<PY
import json
d=json.loads(open('gpurun_out/abv_${v}_c$c.json').read().strip().splitlines()[-1])
print('%-10s c$c'%'$v', 'ms %.3f'%d['ms_per_step'], 'k_split %.3f'%d['roofline']['kernel_ms'], 'mism', d['parity']['mismatches'])
PY
  done
done
