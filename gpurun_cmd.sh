timeout 900 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_bruteforce.py -x -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -2 gpurun_out/t.log
timeout 600 python tools/c1_experiment.py "" "gthr=0" "gthr=1" 2>&1 | tail -3
timeout 600 python tools/stage_experiment.py --opts "gthr=1" > gpurun_out/s.log 2>&1; tail -1 gpurun_out/s.log
timeout 600 python tools/stage_experiment.py --k 100 --nprobe 64 --opts "gthr=1" > gpurun_out/s.log 2>&1; tail -1 gpurun_out/s.log
