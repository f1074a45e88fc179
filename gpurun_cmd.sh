mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "not c2_scale" --timeout 240 -p no:randomly > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
for L in 1 2 3; do timeout 600 python bench.py --lanes $L > gpurun_out/bench_l$L.json 2> gpurun_out/bench_l$L.err; echo bench$L=$?; tail -2 gpurun_out/bench_l$L.err; done
