mkdir -p gpurun_out
timeout 600 python tools/engine_host_profile.py > gpurun_out/eng_host.log 2>&1
