mkdir -p gpurun_out
for o in 0 1; do
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launch_rg$o.csv python tools/c2_profile.py --steps 3 --c3 --opt rerank_group=$o > gpurun_out/c3_ncu_$o.log 2>&1
done
timeout 900 python tools/c3_stages.py "rerank_group=0" "rerank_group=1" "rerank_group=0" "rerank_group=1" > gpurun_out/c3_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_padded.py tests/test_gpu_bruteforce.py -x -q -m gpu > gpurun_out/rg_tests.log 2>&1
