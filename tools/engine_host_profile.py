"""Host-side cost breakdown of the device engine's public API (diagnostic, not a benchmark)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02281_b200 import _lib  # noqa: E402
from paper_2512_02281_b200.ann_graph import VectorStore, build_knn_graph  # noqa: E402
from paper_2512_02281_b200.engine import ContinuousBatchEngine, EngineConfig  # noqa: E402
from paper_2512_02281_b200.workload import gen_matrix  # noqa: E402

data = gen_matrix(100_000, 128, 1)
queries = gen_matrix(4096, 128, 2).astype(np.float64)
store = VectorStore(data=data)
graph = build_knn_graph(store, 16)
eng = ContinuousBatchEngine(store, graph, EngineConfig())
lib = _lib.gpu()
for rep in range(4):
    t1 = time.perf_counter()
    rids = eng.submit_many(queries, 10)
    t2 = time.perf_counter()
    em = np.zeros(4096, np.int64)
    done = C.c_int32(0)
    _lib.check(lib.tri_engine_run(eng._h, 4096, 1, C.byref(done), em.ctypes.data, None, None))
    t3 = time.perf_counter()
    eng._collect()
    t4 = time.perf_counter()
    eng.result_arrays(rids)
    t5 = time.perf_counter()
    ms, n = eng.device_time()
    print(f"submit {1e3*(t2-t1):.2f} run(C) {1e3*(t3-t2):.2f} collect(py) {1e3*(t4-t3):.2f} arrays {1e3*(t5-t4):.2f} "
          f"steps {done.value} device_ms_total {ms:.2f}", flush=True)
