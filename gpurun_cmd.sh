free -g | head -2; nproc
timeout 1500 python tools/bench_c4.py > gpurun_out/c4.log 2> gpurun_out/c4.err; echo c4=$?; tail -6 gpurun_out/c4.log | cut -c1-600; tail -3 gpurun_out/c4.err
