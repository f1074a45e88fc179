mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --full-out gpurun_out/bench_full.json > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
