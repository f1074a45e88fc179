mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_padded.py -q -x > gpurun_out/pytest_pad.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pad.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python tools/c5_realtime.py --repeats 3 --out gpurun_out/c5.json > gpurun_out/c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/c5.log
