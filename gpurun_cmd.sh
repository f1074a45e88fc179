mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ivf.py -x -q -m gpu -k "scan_options" > gpurun_out/opt_tests.log 2>&1
