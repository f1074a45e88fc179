mkdir -p gpurun_out
timeout 1500 python bench.py --full-out gpurun_out/bench_full.json > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
