mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench_sharded.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-configs > gpurun_out/bench.log 2>&1
