mkdir -p gpurun_out
for G in 1 2 4 8; do timeout 900 python tools/bench_c4.py --shards $G --lanes 4 --check 8 --out gpurun_out/c4_G$G.json > gpurun_out/c4_G$G.log 2>&1; done
