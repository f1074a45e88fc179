mkdir -p gpurun_out
for i in 1 2; do timeout 900 python -m pytest tests/test_gpu_stress.py -x -q -m gpu >> gpurun_out/stress2.log 2>&1; done
TRI_GRAPHS=0 timeout 900 python -m pytest tests/test_gpu_stress.py -x -q -m gpu >> gpurun_out/stress2.log 2>&1
