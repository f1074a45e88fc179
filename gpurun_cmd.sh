timeout 900 python bench.py --no-configs > gpurun_out/b.json 2> gpurun_out/b.err; echo bench=$?; python -c "
import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline'];print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['scan_ms_per_launch'],4), r['isolated'])"; tail -2 gpurun_out/b.err
