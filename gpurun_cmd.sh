timeout 600 python tools/stage_experiment.py --opts "scan_qbufs=2" "scan_qbufs=1" "scan_qbufs=2" "scan_qbufs=1" > gpurun_out/s.log 2>&1; tail -4 gpurun_out/s.log
timeout 600 python tools/stage_experiment.py --k 100 --nprobe 64 --opts "scan_qbufs=2" "scan_qbufs=1" > gpurun_out/s2.log 2>&1; tail -2 gpurun_out/s2.log
for q in 2 1; do timeout 600 python bench.py --opt scan_qbufs=$q --cpu-sample 1 --no-configs > gpurun_out/b.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline'];print('qbufs=$q', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['isolated']['frac'],3))"; done
