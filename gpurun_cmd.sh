timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -1 gpurun_out/t.log
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$? secs=$(( $(date +%s) - s )); python -c "
import json;d=json.load(open('gpurun_out/bench_full.json'));r=d['roofline'];print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['isolated']['frac'],3), d['clocks']['samples']); c=d['configs']; print({k:(round(v.get('qps',0)) if isinstance(v,dict) else v) for k,v in c.items()}); print(c['C1']['ms_per_batch'], c['C3']['qps_one_stream'])"
