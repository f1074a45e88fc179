mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -x -q -m gpu > gpurun_out/all_gpu.log 2>&1
timeout 900 python tools/c3_padded.py > gpurun_out/c3_padded.log 2>&1
