# ncu --set full of k_split for a library variant: VARIANT=name NAME=out CONFIG=2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
FPP_LIB=paper_2101_11408_b200/libfpparse_${VARIANT}.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_split -c 1 -s 2 -o gpurun_out/${NAME:-var} python bench.py --config ${CONFIG:-2} --profile-run > gpurun_out/ncu_var.log 2>&1; echo ncu $?
