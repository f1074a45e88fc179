mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:'scan_|merge_|rerank|fixup|prep_|pack_|dense_|finalize|exact_' -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --lanes 1 --cpu-sample 1 > gpurun_out/ncu_b.log 2>&1; echo launches=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:scan_tc_kernel --launch-skip 3 -c 1 -o gpurun_out/scan_full -f python bench.py --steps 2 --warmup 3 --lanes 1 --cpu-sample 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
ls -la gpurun_out
