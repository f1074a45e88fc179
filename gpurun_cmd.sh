mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
TRI_GRAPHS=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/c2_profile.py --steps 2 > gpurun_out/c2_launches.csv 2>&1
rm -f gpurun_out/bench_ab.log
for o in 1 0 1 0; do timeout 600 python bench.py --steps 100 --warmup 5 --no-configs --opt pack_fused=$o > gpurun_out/bench_pf$o.log 2>&1; tail -1 gpurun_out/bench_pf$o.log >> gpurun_out/bench_ab.log; done
