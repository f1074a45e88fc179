mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --full-out gpurun_out/bench_full.json > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --steps 100 --warmup 5 --no-configs --cpu-sample 1 > gpurun_out/b100.log 2>&1
timeout 2400 python -m pytest tests/ -q -m gpu -x > gpurun_out/all_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/all_gpu.log
