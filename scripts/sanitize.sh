# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize.py
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1
python scripts/sanitize.py > gpurun_out/san_plain.log 2>&1; echo plain $?
for tool in memcheck racecheck synccheck; do
  timeout 3000 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo $tool $?; tail -3 gpurun_out/san_$tool.log
done
