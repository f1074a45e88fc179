"""The reference's OWN hot-path tests, run against this package (drop-in proof).

``baseline/ref_tests`` holds the unmodified test files of the reference
(pkg/tests: test_ann_graph.py, test_engine.py, test_scheduler.py,
test_workload.py, test_acceptance.py + conftest.py), copied there by
tools/vendor_reference.sh together with the reference install in
``baseline/_ref`` (both git-ignored, both travel to the GPU box).  The
``trinity_alias`` plugin points ``trinity.ann_graph / engine / scheduler /
workload`` at paper_2512_02281_b200, so every brute-force, distance, graph
build and engine call in those tests runs through libtrinity_b200 on the GPU.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "ref_tests")
FILES = ["test_ann_graph.py", "test_engine.py", "test_scheduler.py", "test_workload.py", "test_acceptance.py"]

# The reference's acceptance criterion 2 is documented by the reference itself
# as failing (its recall ceiling, test_acceptance.py:6-12); nothing else may fail.
KNOWN_REFERENCE_FAILURES = {"test_acceptance.py::test_criterion_2_recall_vs_brute_force"}


@pytest.mark.gpu
def test_reference_suite_passes_against_this_package():
    if not all(os.path.exists(os.path.join(REF_TESTS, f)) for f in FILES):
        pytest.skip("baseline/ref_tests absent: run tools/vendor_reference.sh where /root/reference exists")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), ROOT,
                                                       os.environ.get("PYTHONPATH", "")]))
    cmd = [sys.executable, "-m", "pytest", "-p", "trinity_alias", "-p", "no:cacheprovider", "-q", "-rfE",
           "--rootdir", REF_TESTS, "-c", os.devnull, *[os.path.join(REF_TESTS, f) for f in FILES]]
    res = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1500)
    out = res.stdout + res.stderr
    failed = set(re.findall(r"^(?:FAILED|ERROR) (\S+?)(?: - |$)", out, flags=re.M))
    failed = {f.split("/")[-1] for f in failed}
    assert "passed" in out, out[-3000:]
    assert failed <= KNOWN_REFERENCE_FAILURES, f"reference tests failing against this package: {sorted(failed)}\n" + out[-3000:]
