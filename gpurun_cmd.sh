timeout 1000 python -m pytest tests -m gpu -x -q -k "not c2_scale" --timeout 240 -p no:randomly > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
