mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:randomly > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
for cfg in "2 0" "3 0" "3 16" "3 24" "4 24" "4 32"; do set -- $cfg
timeout 600 python bench.py --lanes $1 --scan-reserve $2 --steps 300 --cpu-sample 1 > gpurun_out/b_$1_$2.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b_$1_$2.json'));r=d['roofline'];print('lanes=$1 reserve=$2', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['scan_ms_per_launch'],4))"; done
