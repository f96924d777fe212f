# numbers for DESIGN.md sections 13-15: binary32 benches, configs 6/7, the Clinger variant A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
B="--steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 python bench.py --dtype f32 $B > gpurun_out/t_f32_c2.json 2>/dev/null
timeout 600 python bench.py --dtype f32 --variant batch $B > gpurun_out/t_f32_c2b.json 2>/dev/null
timeout 600 python bench.py --dtype f32 --config 4 $B > gpurun_out/t_f32_c4.json 2>/dev/null
for c in 2 3 6 7; do
  timeout 600 python bench.py --config $c $B > gpurun_out/t_prod_c$c.json 2>/dev/null
  FPP_LIB=paper_2101_11408_b200/libfpparse_clinger.so timeout 600 python bench.py --config $c $B > gpurun_out/t_cl_c$c.json 2>/dev/null
done
echo done
