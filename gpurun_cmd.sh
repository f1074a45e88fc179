mkdir -p gpurun_out
rm -f gpurun_out/ramp.log
for cfg in "20 4" "20 4" "100 4"; do set -- $cfg
timeout 300 python bench.py --steps $1 --lanes $2 --warmup 5 --no-configs --cpu-sample 1 > gpurun_out/b.log 2>&1; grep '^{' gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps',$1,'lanes',$2, round(d['value']), round(d['ms_per_step']*$1,3), 'e2e', round(d['e2e']['value']))" >> gpurun_out/ramp.log; done
