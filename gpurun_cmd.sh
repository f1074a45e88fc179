mkdir -p gpurun_out
for s in 20 20; do timeout 300 python bench.py --steps $s --warmup 5 --no-configs > gpurun_out/bench_s$s.log 2>&1; grep '^{' gpurun_out/bench_s$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($s, d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step_frac'], d['roofline']['isolated'], d['clocks'])" >> gpurun_out/bench_var.log; done
timeout 900 python bench.py --steps 20 --warmup 5 --full-out gpurun_out/bench_full.json > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
