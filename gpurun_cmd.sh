mkdir -p gpurun_out
timeout 600 python tools/c5_profile.py > gpurun_out/c5_prof.log 2>&1; echo "rc=$?" >> gpurun_out/c5_prof.log
