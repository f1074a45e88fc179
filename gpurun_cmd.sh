export TRI_GRAPHS=0
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'scan_|merge_|rerank|fixup|prep_|pack_|dense_|coarse_' -c 60 --csv --log-file gpurun_out/launches_final2.csv python bench.py --steps 2 --warmup 3 --lanes 1 --cpu-sample 1 --no-configs > /dev/null 2>&1; echo launches=$?
