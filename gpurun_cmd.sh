timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -3 gpurun_out/t.log
timeout 600 python tools/stage_experiment.py --opts "pack_fused=0" "pack_fused=1" > gpurun_out/stage13.log 2>&1; echo exp=$?; cat gpurun_out/stage13.log | tail -2
timeout 600 python tools/c3_stages.py > gpurun_out/c3.log 2>&1; echo c3=$?; tail -1 gpurun_out/c3.log
for L in 3; do timeout 600 python bench.py --lanes $L --steps 300 --cpu-sample 1 --no-configs > gpurun_out/b.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline'];print('lanes=$L', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['scan_ms_per_launch'],4))"; done
