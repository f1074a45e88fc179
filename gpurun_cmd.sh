timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_engine_device.py tests/test_gpu_bruteforce.py -x -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -2 gpurun_out/t.log
timeout 600 python tools/bench_engine.py > gpurun_out/eng1.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/eng1.json')); print({k: d[k] for k in ('qps','us_per_step','parity')})"
timeout 600 python tools/bench_engine.py --n 20000 --d 768 --nq 1024 > gpurun_out/eng2.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/eng2.json')); print({k: d[k] for k in ('qps','us_per_step','parity')})"
