# Round measurement pass: smoke, GPU tests, bench lines for every config and
# variant, ncu launch lists (C2, C5) and --set full captures of the dominant
# kernels, summarised on the box (reports are ~25 MB; gpurun copies back at
# most 64 MiB).  Outputs under gpurun_out/fin_*.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/fin_pytest.log 2>&1; echo pytest $?
timeout 900 python bench.py > gpurun_out/fin_bench_c2.json 2> gpurun_out/fin_bench_c2.err; echo bench $?
for c in 3 4 5 6 7 8; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/fin_bench_c$c.json 2>gpurun_out/fin_bench_c$c.err; done
timeout 600 python bench.py --variant batch --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/fin_bench_c2_batch.json 2>gpurun_out/fin_bench_c2_batch.err
timeout 600 python bench.py --dtype f32 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/fin_bench_c2_f32.json 2>gpurun_out/fin_bench_c2_f32.err
timeout 600 python bench.py --grammar json --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fin_bench_c2_json.json 2>gpurun_out/fin_bench_c2_json.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_ref.json 2>gpurun_out/fin_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches_c2.csv python bench.py --profile-run > gpurun_out/fin_ncu_launch2.log 2>&1; echo ncu1 $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches_c5.csv python bench.py --config 5 --profile-run > gpurun_out/fin_ncu_launch5.log 2>&1; echo ncu5 $?
KERNEL=k_split CFG=2 TAG=fin_c2_split RECS=100000000 KEEP=1 bash scripts/ncu_sum.sh
KERNEL=k_batch CFG=2 TAG=fin_c2_batch RECS=100000000 ARGS="--variant batch" bash scripts/ncu_sum.sh
KERNEL="^k_slow$" CFG=5 TAG=fin_c5_slow RECS=7450000 bash scripts/ncu_sum.sh
KERNEL=k_slow_scan CFG=5 TAG=fin_c5_scan RECS=10000000 bash scripts/ncu_sum.sh
cp profiles/ncu_summary.json gpurun_out/fin_ncu_summary.json
