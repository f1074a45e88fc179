timeout 900 python -m pytest tests -m gpu -x -q -k "not c2_scale" > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
python tools/scan_experiment.py --modes 0,1,3 --kernels 0 2>&1 | tail -3
