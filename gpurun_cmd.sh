mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
for o in 1 0 1 0; do timeout 600 python bench.py --steps 100 --warmup 5 --no-configs --opt coarse_set=$o > gpurun_out/bench_cs$o.log 2>&1; tail -1 gpurun_out/bench_cs$o.log >> gpurun_out/bench_ab.log; done
