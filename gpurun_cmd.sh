mkdir -p gpurun_out
for i in 1 2; do
BENCH_DEVICE=0 BENCH_BACKEND=gloo BENCH_C4_N=300000 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$i bench.py --gpus 2 --steps 4 --warmup 3 --lanes 2 --parity full > gpurun_out/sh$i.out 2> gpurun_out/sh$i.err; echo "rc=$?" >> gpurun_out/sh$i.err
done
