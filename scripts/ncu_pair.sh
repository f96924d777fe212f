# ncu --set full of k_split on several configs: CONFIGS="2 4" TAG=name [FPP_LIB=...]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
for c in ${CONFIGS:-2}; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_split} -c 1 -s 2 -o gpurun_out/${TAG}_c$c python bench.py --config $c --profile-run ${ARGS} > gpurun_out/ncu_${TAG}_c$c.log 2>&1; echo ncu c$c $?
done
