# time library variants on config 2 (and others in $CONFIGS): FPP_LIB=<variant .so>
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1
for v in product ${VARIANTS}; do
  lib=""; [ "$v" != product ] && lib=paper_2101_11408_b200/libfpparse_$v.so
  for c in ${CONFIGS:-2}; do
    FPP_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/v_${v}_c$c.json 2>gpurun_out/v_${v}_c$c.err
    python - <<PY
import json
d=json.loads(open('gpurun_out/v_${v}_c$c.json').read().strip().splitlines()[-1])
print('$v c$c', 'ms %.3f'%d['ms_per_step'], 'kern %.3f'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'], 'mism', d['parity']['mismatches'], 'mhz', d['clocks']['sm_mhz'])
PY
  done
done
