mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_bruteforce.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
TRI_GRAPHS=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/c2_profile.py --steps 2 > gpurun_out/c2_launches.csv 2>&1
rm -f gpurun_out/bench_ab.log
for o in 1 0 1 0; do timeout 600 python bench.py --steps 100 --warmup 5 --no-configs --opt rerank_oneslab=$o 2>/dev/null | tail -1 >> gpurun_out/bench_ab.log; done
timeout 300 python tools/c1_experiment.py "rerank_oneslab=1" "rerank_oneslab=0" "rerank_oneslab=1" > gpurun_out/c1.log 2>&1
