mkdir -p gpurun_out
timeout 1500 python bench.py --full-out gpurun_out/bench_full.json > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launches.csv python tools/c2_profile.py --steps 3 > gpurun_out/c2_ncu.log 2>&1
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_c3_launches.csv python tools/c2_profile.py --steps 3 --c3 > gpurun_out/c3_ncu.log 2>&1
