# A/B on one box: parity tests, then VARIANTS (prebuilt libfpparse_<v>.so) vs the product on CONFIGS; NCU=name: one capture of the product
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1 || { echo build failed; tail gpurun_out/ab_build.log; exit 1; }
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest $?; tail -2 gpurun_out/ab_pytest.log; fi
for c in ${CONFIGS:-2}; do
  for v in product ${VARIANTS}; do
    lib=""; [ "$v" != product ] && lib=paper_2101_11408_b200/libfpparse_$v.so
    FPP_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS} > gpurun_out/ab_${v}_c$c.json 2>gpurun_out/ab_${v}_c$c.err
    python - <<PY
import json
d=json.loads(open('gpurun_out/ab_${v}_c$c.json').read().strip().splitlines()[-1])
print('%-10s c$c'%'$v', 'ms %.3f'%d['ms_per_step'], 'kern %.3f'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'], 'mism', d['parity']['mismatches'], 'mhz', d['clocks']['sm_mhz'])
PY
  done
done
if [ -n "$NCU" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_split -c 1 -s 2 -o gpurun_out/$NCU python bench.py --profile-run ${BENCH_ARGS} > gpurun_out/ab_ncu.log 2>&1; echo ncu $?
fi
