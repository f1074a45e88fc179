timeout 900 python -m pytest tests -m gpu -x -q -k "not c2_scale" > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/gpu_tests.log
python tools/scan_experiment.py --modes 0 --kernels 0 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bf_launches.csv python tools/bf_experiment.py 0 1 > /dev/null 2>&1; echo ncu=$?
