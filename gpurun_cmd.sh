mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_ivf.py -q -x -k "c4_scale" > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
