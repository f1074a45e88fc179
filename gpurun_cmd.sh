timeout 900 python -m pytest tests -m gpu -x -q -k "not c2_scale" > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -25 gpurun_out/gpu_tests.log
