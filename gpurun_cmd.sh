mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/all_gpu.log 2>&1
TRI_GRAPHS=0 timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
TRI_GRAPHS=0 timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
TRI_GRAPHS=0 timeout 1500 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
