mkdir -p gpurun_out
for o in 0 1; do
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launch_gb$o.csv python tools/c2_profile.py --steps 3 --c3 --opt merge_gb=$o > gpurun_out/c3_ncu.log 2>&1
done
timeout 900 python tools/c3_stages.py "merge_gb=0" "merge_gb=1" "merge_gb=0" "merge_gb=1" > gpurun_out/c3_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_padded.py -x -q -m gpu > gpurun_out/gb_tests.log 2>&1
