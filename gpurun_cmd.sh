mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_engine_device.py -x -q --timeout 600 -p no:randomly > gpurun_out/eng_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/eng_tests.log
timeout 600 python tools/bench_engine.py > gpurun_out/eng1.json 2>gpurun_out/eng1.err; echo e1=$?; cat gpurun_out/eng1.json; tail -3 gpurun_out/eng1.err
timeout 600 python tools/bench_engine.py --n 20000 --d 768 --nq 1024 > gpurun_out/eng2.json 2>gpurun_out/eng2.err; echo e2=$?; cat gpurun_out/eng2.json; tail -3 gpurun_out/eng2.err
