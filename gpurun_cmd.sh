mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_engine_device.py -x -q --timeout 600 -p no:randomly > gpurun_out/eng_tests.log 2>&1; echo tests=$?; tail -30 gpurun_out/eng_tests.log
