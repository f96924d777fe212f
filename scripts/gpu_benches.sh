# smoke, gpu tests, benches (all configs, batch, f32, grammar) -- no ncu (gpurun_out stays small)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench $?
for c in 3 4 5 6 7 8; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; done
timeout 600 python bench.py --variant batch --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_batch.json 2>gpurun_out/bench_c2_batch.err
timeout 600 python bench.py --dtype f32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_f32.json 2>gpurun_out/bench_c2_f32.err
timeout 600 python bench.py --grammar json --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c2_json.json 2>gpurun_out/bench_c2_json.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile-run > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --config 5 --profile-run > gpurun_out/ncu_launch5.log 2>&1; echo ncu5 $?
