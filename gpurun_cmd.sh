mkdir -p gpurun_out
TRI_GRAPHS=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scan_tc --launch-skip 50 -c 3 --csv python tools/c1_experiment.py 2>/dev/null | grep scan_tc | awk -F'","' '{print "c1", $NF}' > gpurun_out/ins.log
TRI_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scan_tc --launch-skip 20 -c 2 --csv python tools/c3_fixups.py 2>/dev/null | grep scan_tc | awk -F'","' '{print "c3", $NF}' >> gpurun_out/ins.log
timeout 300 python tools/stage_experiment.py --opts "" "" >> gpurun_out/ins.log 2>&1
