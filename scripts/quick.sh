# quick GPU iteration: parity tests + short benches (no cpu baseline / e2e)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1 || { echo build failed; tail gpurun_out/q_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo pytest $?; tail -3 gpurun_out/q_pytest.log
for c in ${CONFIGS:-2 3 4}; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q_c$c.json 2>gpurun_out/q_c$c.err
  python - <<PY
import json
d=json.loads(open('gpurun_out/q_c$c.json').read().strip().splitlines()[-1])
print('c$c', 'ms %.3f'%d['ms_per_step'], 'kern %.3f'%d['roofline']['kernel_ms'], 'GB/s %.1f'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'mism', d['parity']['mismatches'], 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
done
if [ -n "$NCU" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_split -c 1 -s 2 -o gpurun_out/$NCU python bench.py --profile-run > gpurun_out/q_ncu.log 2>&1; echo ncu $?
fi
if [ -n "$BATCH" ]; then
  timeout 600 python bench.py --variant batch --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q_batch.json 2>gpurun_out/q_batch.err
  python -c "
import json
d=json.loads(open('gpurun_out/q_batch.json').read().strip().splitlines()[-1])
print('batch c2', 'ms %.3f'%d['ms_per_step'], 'kern %.3f'%d['roofline']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'], 'mism', d['parity']['mismatches'])"
fi
