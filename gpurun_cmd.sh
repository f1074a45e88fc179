mkdir -p gpurun_out
timeout 600 python tools/dense_ab.py --option scan_qbufs --values 2,3 > gpurun_out/qb3_ab.log 2>&1
timeout 900 python tools/c3_stages.py "scan_qbufs=2" "scan_qbufs=3" "scan_qbufs=2" "scan_qbufs=3" > gpurun_out/c3_qb3.log 2>&1
