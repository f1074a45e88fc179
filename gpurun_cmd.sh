mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
export TRI_GRAPHS=0
$NCU --metrics gpu__time_duration.sum --clock-control none -k regex:'scan_|merge_|rerank|fixup|prep_|pack_|dense_' -c 60 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --lanes 1 --cpu-sample 1 --no-configs > gpurun_out/ncu_b.log 2>&1; echo launches=$?
$NCU --set full --clock-control none --import-source on -k regex:'scan_tc_kernel|dense_gemm|dense_select|rerank_fused' --launch-skip 12 -c 4 -o gpurun_out/final_full -f python bench.py --steps 2 --warmup 3 --lanes 1 --cpu-sample 1 --no-configs > gpurun_out/ncu_full.log 2>&1; echo full=$?
