s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$? secs=$(( $(date +%s) - s )); python -c "
import json;d=json.load(open('gpurun_out/bench_full.json'));r=d['roofline'];print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['isolated']['frac'],3), d['gpu_launches'], d['clocks'], d['e2e']['batch_latency_ms']['p99'])"
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref=$? secs=$(( $(date +%s) - s )); python -c "
import json;d=json.load(open('gpurun_out/ref.json')); print(d['value'], d['cpu_baseline'])"
