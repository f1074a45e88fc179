timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -1 gpurun_out/t.log
timeout 600 python tools/stage_experiment.py --opts "dense_pow2=1" "dense_pow2=0" "dense_pow2=1" "dense_pow2=0" > gpurun_out/s.log 2>&1; tail -4 gpurun_out/s.log
timeout 600 python tools/stage_experiment.py --k 100 --nprobe 64 --opts "dense_pow2=1" "dense_pow2=0" > gpurun_out/s2.log 2>&1; tail -2 gpurun_out/s2.log
