import sys, json, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import bench_configs as b
from oracle import trinity_oracle as orc
from paper_2512_02281_b200.ann_graph import _DeviceStore
from paper_2512_02281_b200.ivf import IVFFlatIndex
from paper_2512_02281_b200.workload import gen_vectors_chunked
data = gen_vectors_chunked(1_000_000, 768, 3)
idx = IVFFlatIndex.train(_DeviceStore(data), 1024, 5, 4)
cen, asg = idx.export()
art = orc.IVFArtifact(cen, asg)
idx.set_profiling(True)
print(json.dumps(b.c3(idx, data, art, n_requests=int(sys.argv[1]) if len(sys.argv) > 1 else 1200)))
st, n = idx.stage_times()
print({k: round(v / n * 1e3, 1) for k, v in st.items()}, n)
