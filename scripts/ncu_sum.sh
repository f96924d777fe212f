# ncu --set full of one kernel, summarised ON THE BOX (reports are ~25 MB;
# gpurun copies back at most 64 MiB): KERNEL=regex CFG=n TAG=name RECS=n [ARGS=...] [KEEP=1]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KERNEL} -c 1 -s ${SKIP:-2} -o gpurun_out/${TAG} python bench.py --config ${CFG:-2} --profile-run ${ARGS} > gpurun_out/ncu_${TAG}.log 2>&1; echo ncu $?
python profiles/summarize.py full gpurun_out/${TAG}.ncu-rep ${RECS:-100000000} ${TAG} > gpurun_out/${TAG}_sum.md 2>&1
python profiles/summarize.py lines gpurun_out/${TAG}.ncu-rep ${RECS:-100000000} > gpurun_out/${TAG}_lines.md 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
[ -z "$KEEP" ] && rm -f gpurun_out/${TAG}.ncu-rep
ls -la gpurun_out/${TAG}*
