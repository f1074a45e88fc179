mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "not c2_scale" --timeout 240 -p no:randomly > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -4 gpurun_out/gpu_tests.log
timeout 600 python tools/scan_experiment.py --kernels 0,2 --modes 0,1 > gpurun_out/scan_exp.log 2>&1; echo exp=$?; cat gpurun_out/scan_exp.log | tail -4
for L in 1 3; do timeout 600 python bench.py --lanes $L > gpurun_out/bench_l$L.json 2> gpurun_out/bench_l$L.err; echo bench$L=$?; tail -2 gpurun_out/bench_l$L.err; done
