# one ncu --set full capture: KERNEL=k_split|k_batch|k_slow ARGS="bench args" OUT=name
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KERNEL} -c 1 -s ${SKIP:-2} -o gpurun_out/${OUT} python bench.py ${ARGS} --profile-run > gpurun_out/ncu_${OUT}.log 2>&1; echo ncu $?
ls -la gpurun_out/${OUT}.ncu-rep
