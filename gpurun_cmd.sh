mkdir -p gpurun_out
timeout 900 python tools/bench_engine.py --n 2000000 --d 128 --nq 4096 --reps 3 --graph random > gpurun_out/engine_hbm.json 2> gpurun_out/engine_hbm.err
timeout 900 python tools/bench_engine.py --n 100000 --d 128 --nq 4096 --reps 3 --graph random > gpurun_out/engine_l2_random.json 2>> gpurun_out/engine_hbm.err
TRI_GRAPHS=0 timeout 900 ncu --set full --clock-control none -k regex:engine_step -s 5 -c 1 -o gpurun_out/engine_hbm python tools/bench_engine.py --n 2000000 --d 128 --nq 4096 --reps 1 --graph random > gpurun_out/engine_ncu.log 2>&1
