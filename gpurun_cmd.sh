mkdir -p gpurun_out
timeout 120 python tools/c1_scan_probe.py scan_debug=8 20 > gpurun_out/c1_ts.log 2>&1
timeout 300 python tools/c1_experiment.py "" "bf_wide=0" > gpurun_out/c1.log 2>&1
TRI_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 400 -c 7 --csv python tools/c1_experiment.py > gpurun_out/c1_launches.csv 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
