timeout 600 python tools/c3_stages.py "" > gpurun_out/c3.log 2>&1; tail -1 gpurun_out/c3.log | cut -c1-200
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?; python -c "
import json;d=json.load(open('gpurun_out/bench_full.json'));r=d['roofline'];print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['isolated']['frac'],3)); c=d['configs']; print(json.dumps(c['C3'])[:600])"
