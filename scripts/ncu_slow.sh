mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_slow -c 1 -s 1 -o gpurun_out/${NAME:-slow} python bench.py --config 5 --profile-run > gpurun_out/ncu_slow.log 2>&1; echo ncu $?
