timeout 300 python -c "
import sys, json; sys.path.insert(0,'tools'); import bench_configs as b; r=b.c1(); print(r['qps'], r['ms_per_batch'], r['parity'], json.dumps(r['batch_sweep']))"
