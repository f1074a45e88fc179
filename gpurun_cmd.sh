mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "not c2_scale" --timeout 240 -p no:randomly > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 600 python tools/scan_experiment.py --kernels 0,2 --modes 0,1,3 > gpurun_out/scan_exp.log 2>&1; echo exp=$?; tail -6 gpurun_out/scan_exp.log
for L in 1 2 3; do timeout 600 python bench.py --lanes $L > gpurun_out/bench_l$L.json 2> gpurun_out/bench_l$L.err; echo bench=$?; python -c "
import json;d=json.load(open('gpurun_out/bench_l$L.json'));r=d['roofline'];print('l$L', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['scan_ms_per_launch'],4))"; done
