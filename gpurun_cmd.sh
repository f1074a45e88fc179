timeout 900 python -m pytest tests/test_gpu_ivf.py -x -q --timeout 600 -p no:randomly -k "c3_scale or c2_scale" > gpurun_out/t.log 2>&1; echo tests=$?; tail -3 gpurun_out/t.log
