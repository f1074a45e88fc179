"""pytest plugin: ``trinity`` (the reference package) with its hot-path
modules replaced by this repo's B200 implementations.

``trinity.ann_graph``, ``trinity.engine``, ``trinity.scheduler`` and
``trinity.workload`` resolve to ``paper_2512_02281_b200``'s modules, exactly
what a maintainer's drop-in would do; the out-of-scope
modules (cluster_sim, config, report, roofline, ...) stay the reference's own,
loaded from ``baseline/_ref`` (tools/vendor_reference.sh).  Used by
tests/test_gpu_reference_suite.py as ``python -m pytest -p trinity_alias``.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2512_02281_b200 import ann_graph, engine, scheduler, workload  # noqa: E402

for _name, _mod in (("ann_graph", ann_graph), ("engine", engine), ("scheduler", scheduler),
                    ("workload", workload)):
    sys.modules["trinity." + _name] = _mod

import trinity  # noqa: E402  (the reference __init__, importing the aliased modules)

for _name in ("ann_graph", "engine", "scheduler", "workload"):
    setattr(trinity, _name, sys.modules["trinity." + _name])
    assert sys.modules["trinity." + _name].__name__.startswith("paper_2512_02281_b200")
