timeout 600 python tools/_srch_tmp.py 2>&1 | tail -4
