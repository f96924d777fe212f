# ncu --set full captures of the three kernels (one .ncu-rep each)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_split -c 1 -s 2 -o gpurun_out/full_c2_split python bench.py --profile-run > gpurun_out/ncu_full.log 2>&1; echo ncu2 $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_batch -c 1 -s 2 -o gpurun_out/full_c2_batch python bench.py --variant batch --profile-run > gpurun_out/ncu_full_b.log 2>&1; echo ncu3 $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_slow -c 1 -s 1 -o gpurun_out/full_c5_slow python bench.py --config 5 --profile-run > gpurun_out/ncu_full_s.log 2>&1; echo ncu4 $?
