mkdir -p gpurun_out
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$? secs=$(( $(date +%s) - s )); cat gpurun_out/bench_full.json; tail -5 gpurun_out/bench_full.err
