mkdir -p gpurun_out
timeout 900 python tools/c3_stages.py "" "" "" "" > gpurun_out/c3_e2e.log 2>&1
