mkdir -p gpurun_out
timeout 900 python tools/c5_realtime.py --repeats 3 --out gpurun_out/c5.json > gpurun_out/c5.log 2>&1; echo "rc=$?" >> gpurun_out/c5.log
timeout 900 python -m pytest tests/test_gpu_pool.py -q -x > gpurun_out/pool_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pool_gpu.log
