for cfg in "3 0" "3 8" "3 12" "3 16" "4 0" "4 8" "4 16"; do set -- $cfg
timeout 600 python bench.py --lanes $1 --scan-reserve $2 --steps 300 --cpu-sample 1 --no-configs > gpurun_out/b.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline'];print('lanes=$1 reserve=$2', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), round(r['frac'],3), round(r['isolated']['frac'],3))"; done
