timeout 600 python tools/bench_engine.py > gpurun_out/eng1.json 2>gpurun_out/eng1.err; echo e1=$?; python -c "
import json; d=json.load(open('gpurun_out/eng1.json')); print({k: d[k] for k in ('qps','e2e_batched_qps','sequential_qps','sequential_device_qps','batch_fill','parity')})"; tail -2 gpurun_out/eng1.err
