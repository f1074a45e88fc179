mkdir -p gpurun_out
rm -f gpurun_out/ramp.log
for cfg in "20 -1" "20 -1" "100 -1"; do set -- $cfg
timeout 300 python bench.py --steps $1 --warmup 5 --no-configs --cpu-sample 1 --scan-reserve $2 > gpurun_out/b.log 2>&1; grep '^{' gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps',$1,'res',$2, round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3))" >> gpurun_out/ramp.log; done
timeout 900 python bench.py --steps 20 --warmup 5 --full-out gpurun_out/bench_full.json > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
