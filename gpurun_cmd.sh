mkdir -p gpurun_out
timeout 600 python -c "
import sys, json; sys.path.insert(0,'.'); sys.path.insert(0,'tools')
import bench, bench_configs as bc
r = bc.c1(bench.load_peaks()[0]); print(json.dumps({k: r[k] for k in ('value','e2e','parity')}))
" > gpurun_out/c1cfg.log 2>&1
