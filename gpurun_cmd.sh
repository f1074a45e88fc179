mkdir -p gpurun_out
cd baseline/ref_tests && PYTHONPATH=../../tests:../..:$PYTHONPATH timeout 900 python -m pytest -p trinity_alias -p no:cacheprovider -q -rfE --rootdir . -c /dev/null test_ann_graph.py test_engine.py test_scheduler.py test_workload.py test_acceptance.py > ../../gpurun_out/refsuite_full.log 2>&1; echo "rc=$?" >> ../../gpurun_out/refsuite_full.log
