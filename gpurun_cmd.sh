mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_padded.py tests/test_gpu_ivf.py tests/test_gpu_bruteforce.py tests/test_gpu_pool.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
timeout 900 python tools/c3_padded.py > gpurun_out/c3p.log 2>&1; echo "rc=$?" >> gpurun_out/c3p.log
