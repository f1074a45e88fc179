mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
start=$(date +%s)
timeout 1200 python bench.py --steps 20 --warmup 5 --full-out gpurun_out/full.json > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.log 2> gpurun_out/ref.err; echo "ref rc=$?" >> gpurun_out/ref.err
