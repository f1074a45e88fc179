mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_torch_ops.py tests/test_gpu_bruteforce.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
