mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bruteforce.py tests/test_gpu_padded.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
start=$(date +%s)
timeout 1200 python bench.py --steps 20 --warmup 5 --full-out gpurun_out/full.json > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s" >> gpurun_out/bench.err
