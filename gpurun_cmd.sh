mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  TRI_GRAPHS=0 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
done
