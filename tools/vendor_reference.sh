#!/bin/bash
# Run HERE (the container that has /root/reference): install the unmodified
# reference into baseline/_ref (its own pip build, --no-deps) and copy its
# hot-path test files into baseline/ref_tests/.  Both directories are
# git-ignored (reference sources never enter this repo's history) but travel
# to the GPU box with gpurun, where tests/test_gpu_reference_suite.py runs the
# reference's own tests with `trinity` pointing at this package.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target "$ROOT/baseline/_ref" --upgrade "$TMP/ref/pkg" > /dev/null
mkdir -p "$ROOT/baseline/ref_tests"
for f in conftest.py test_ann_graph.py test_engine.py test_scheduler.py test_workload.py test_acceptance.py; do
  cp "$TMP/ref/pkg/tests/$f" "$ROOT/baseline/ref_tests/$f"
done
cp "$TMP/ref/pkg/test_output.txt" "$ROOT/baseline/ref_tests/test_output.txt"
rm -rf "$TMP"
echo "reference installed in baseline/_ref, tests in baseline/ref_tests"
