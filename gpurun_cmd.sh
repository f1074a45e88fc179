mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_engine_device.py -x -q --timeout 600 -p no:randomly > gpurun_out/eng_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/eng_tests.log
timeout 600 python tools/engine_host_profile.py 2>&1 | tail -3
timeout 600 python tools/bench_engine.py > gpurun_out/eng1.json 2>gpurun_out/eng1.err; echo e1=$?; python -c "
import json; d=json.load(open('gpurun_out/eng1.json')); print({k: d[k] for k in ('qps','us_per_step','e2e_qps','e2e_batched_qps','parity','steps')})"; tail -3 gpurun_out/eng1.err
