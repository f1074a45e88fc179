timeout 900 python -m pytest tests/test_gpu_ivf.py -x -q --timeout 600 -p no:randomly -k duplicate > gpurun_out/t.log 2>&1; echo tests=$?; tail -15 gpurun_out/t.log
