#!/bin/bash
# build here (fail fast), then run gpurun_cmd.sh on the B200 box
python -c "from paper_2512_02281_b200 import _build; _build.build()" > /tmp/build.log 2>&1 || { echo "BUILD FAILED"; grep -m5 error /tmp/build.log; exit 1; }
/usr/local/graft/bin/gpurun --timeout ${1:-1800} -- 'bash gpurun_cmd.sh' > /tmp/gpurun_last.log 2>&1
tail -1 /tmp/gpurun_last.log
