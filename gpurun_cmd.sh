mkdir -p gpurun_out
timeout 600 python tools/dense_ab.py --option scan_pool_minkp --values 128,32 > gpurun_out/dense_ab.log 2>&1
for o in 128 32; do
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launch_mk$o.csv python tools/c2_profile.py --steps 3 --opt scan_pool_minkp=$o > gpurun_out/c2_ncu.log 2>&1
timeout 300 python tools/c2_profile.py --steps 3 --opt scan_debug=16,scan_pool_minkp=$o > gpurun_out/c2_cnt_$o.log 2>&1
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launch_mk$o.csv python tools/c2_profile.py --steps 3 --c3 --opt scan_pool_minkp=$o > gpurun_out/c3_ncu.log 2>&1
done
