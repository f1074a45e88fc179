timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -2 gpurun_out/t.log
timeout 600 python tools/stage_experiment.py --opts "coarse_tc=1" > gpurun_out/s.log 2>&1; tail -1 gpurun_out/s.log
