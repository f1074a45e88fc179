mkdir -p gpurun_out
for o in 0 1 2 4; do
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launch_pf$o.csv python tools/c2_profile.py --steps 3 --c3 --opt pack_first=$o > gpurun_out/c3_ncu.log 2>&1
timeout 300 python tools/c2_profile.py --steps 3 --c3 --opt scan_debug=16,pack_first=$o > gpurun_out/c3_cnt_$o.log 2>&1
done
timeout 900 python tools/c3_stages.py "pack_first=0" "pack_first=2" "pack_first=0" "pack_first=2" > gpurun_out/c3_ab.log 2>&1
