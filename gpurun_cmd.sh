mkdir -p gpurun_out
timeout 900 python tools/c3_stages.py "merge_split=0" "merge_split=1" "merge_split=0" "merge_split=1" > gpurun_out/c3_ms.log 2>&1
TRI_GRAPHS=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/c2_profile.py --steps 3 --c3 > gpurun_out/c3_ncu.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_padded.py tests/test_gpu_pool.py tests/test_gpu_stress.py tests/test_gpu_bruteforce.py -q -x > gpurun_out/ms_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ms_tests.log
