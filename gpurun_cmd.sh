timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:randomly > gpurun_out/t.log 2>&1; echo tests=$?; tail -2 gpurun_out/t.log
export TRI_GRAPHS=0
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'dense_select' -c 10 --csv --log-file gpurun_out/sel2.csv python tools/stage_experiment.py --n 300000 > /dev/null 2>&1; echo ncu=$?
