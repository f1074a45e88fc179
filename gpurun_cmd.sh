mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_sharded.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
