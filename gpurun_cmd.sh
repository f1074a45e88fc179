mkdir -p gpurun_out
timeout 300 python tools/c1_experiment.py "" "" > gpurun_out/c1.log 2>&1
TRI_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 -c 8 --csv python tools/c1_experiment.py > gpurun_out/c1_launches.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_bruteforce.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
