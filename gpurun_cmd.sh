mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
cd baseline/ref_tests && PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT timeout 900 python -m pytest -p trinity_alias -p no:cacheprovider -rA --rootdir . -c /dev/null test_ann_graph.py test_engine.py test_scheduler.py test_workload.py test_acceptance.py > $GRAFT_REPO_ROOT/gpurun_out/refsuite_full.log 2>&1; echo "rc=$?" >> $GRAFT_REPO_ROOT/gpurun_out/refsuite_full.log
