mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -3 gpurun_out/t.log
timeout 600 python tools/stage_experiment.py --opts "force_fixup=1" "force_fixup=0" > gpurun_out/stage12.log 2>&1; echo exp=$?; cat gpurun_out/stage12.log | tail -2
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?; python -c "
import json;d=json.load(open('gpurun_out/bench_full.json'));r=d['roofline'];print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['scan_ms_per_launch'],4)); c=d['configs']; print({k:(round(v.get('qps',0)) if isinstance(v,dict) else v) for k,v in c.items()}); print(c['C3'].get('parity'), c['C1'].get('parity'), c['engine'].get('parity'))"
