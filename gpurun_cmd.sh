timeout 600 python tools/c1_experiment.py "bf_f16=1" "bf_f16=0" "bf_f16=1" "bf_f16=0" "bf_f16=1" "bf_f16=0" 2>&1 | tail -6
