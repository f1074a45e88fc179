mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine_device.py tests/test_gpu_engine.py tests/test_gpu_reference_suite.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
timeout 900 python tools/bench_engine.py --n 100000 --d 128 --nq 4096 --reps 3 > gpurun_out/engine_l2.json 2> gpurun_out/engine.err
