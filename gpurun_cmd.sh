mkdir -p gpurun_out
cat > /tmp/eng_ab.py <<'PY'
import sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
from bench_engine import run
from paper_2512_02281_b200 import _lib
for n, kind in [(100_000, "knn"), (2_000_000, "random")]:
    for v in [0, 1, 0, 1]:
        _lib.set_option("eng_prefetch", v)
        r = run(n=n, graph_kind=kind, reps=3, cpu_sample=2)
        print(n, kind, "prefetch", v, {k: r[k] for k in r if k in ("value", "parity")}, json.dumps(r.get("roofline", {}))[:160], flush=True)
PY
timeout 1200 python /tmp/eng_ab.py > gpurun_out/eng_ab.log 2>&1; echo "rc=$?" >> gpurun_out/eng_ab.log
