mkdir -p gpurun_out
timeout 900 python tools/c3_stages.py "rerank_split=0" "rerank_split=1" "rerank_split=0" "rerank_split=1" > gpurun_out/c3_split.log 2>&1
timeout 2400 python -m pytest tests/ -q -m gpu -x > gpurun_out/all_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/all_gpu.log
