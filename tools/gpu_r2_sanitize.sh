# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py
mkdir -p gpurun_out/r2
python tools/sanitize.py > gpurun_out/r2/san_plain.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/r2/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2/san_$tool.log
done
