mkdir -p gpurun_out
BENCH_DEVICE=0 BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --cpu-sample 1 > gpurun_out/b2.json 2> gpurun_out/b2.err; echo b2=$?; cat gpurun_out/b2.json; tail -20 gpurun_out/b2.err
