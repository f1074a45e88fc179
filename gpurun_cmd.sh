mkdir -p gpurun_out
timeout 900 python tools/c3_stages.py "fold_own=1" "fold_own=0" "fold_own=1" "fold_own=0" > gpurun_out/c3s.log 2>&1
