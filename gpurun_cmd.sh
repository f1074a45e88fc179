mkdir -p gpurun_out
TRI_GRAPHS=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/c2_profile.py --steps 3 > gpurun_out/c2_launches.csv 2>&1
TRI_GRAPHS=0 timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:scan_tc -c 1 -o gpurun_out/c2_scan python tools/c2_profile.py --steps 1 > gpurun_out/c2_ncu.log 2>&1
TRI_GRAPHS=0 timeout 1200 ncu --profile-from-start off --set full --clock-control none -c 12 -o gpurun_out/c2_step python tools/c2_profile.py --steps 1 > gpurun_out/c2_ncu_step.log 2>&1
