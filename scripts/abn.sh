# A/B timing (product vs VARIANTS) on CONFIGS, then ncu --set full of the product's k_split on NCU_CONFIGS
# (saves the product cubin next to the reports for offline line attribution)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1 || { echo build failed; tail gpurun_out/ab_build.log; exit 1; }
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q $TESTS > gpurun_out/ab_pytest.log 2>&1; echo pytest $?; tail -2 gpurun_out/ab_pytest.log; fi
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
for c in ${NCU_CONFIGS}; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_split -c 1 -s 2 -o gpurun_out/${TAG:-p}_c$c python bench.py --config $c --profile-run > gpurun_out/ncu_${TAG:-p}_c$c.log 2>&1; echo ncu c$c $?
done
