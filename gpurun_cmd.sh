timeout 300 python tools/_dbg_saveload.py
