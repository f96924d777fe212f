# Round measurement pass: smoke, GPU tests, bench lines for every config and
# variant, ncu launch lists (C2, C5) and --set full captures of the dominant
# kernels.  Outputs under gpurun_out/fin_*; summaries go to profiles/ (here).
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
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_split -c 1 -s 2 -o gpurun_out/fin_c2_split python bench.py --profile-run > gpurun_out/fin_ncu_c2.log 2>&1; echo ncuf2 $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_batch -c 1 -s 2 -o gpurun_out/fin_c2_batch python bench.py --variant batch --profile-run > gpurun_out/fin_ncu_c2b.log 2>&1; echo ncuf2b $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_slow -c 1 -s 2 -o gpurun_out/fin_c5_slow python bench.py --config 5 --profile-run > gpurun_out/fin_ncu_c5.log 2>&1; echo ncuf5 $?
