mkdir -p gpurun_out
for i in 1 2; do timeout 900 python bench.py --steps 20 --warmup 5 --configs C3,C5 --full-out gpurun_out/bf$i.json > gpurun_out/b$i.log 2>&1; done
