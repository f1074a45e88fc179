mkdir -p gpurun_out
timeout 600 python tools/c1_experiment.py "" "gthr=0" "gthr=1,tc_box_rows=32" "tc_box_rows=64" "tc_box_rows=128,tc_stages=4" "tc_stages=0,scan_kernel=1" "scan_kernel=0,dense_off=0" > gpurun_out/c1x.log 2>&1; echo x=$?; cat gpurun_out/c1x.log | tail -8
