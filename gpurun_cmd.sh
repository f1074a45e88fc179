mkdir -p gpurun_out
for o in 0 128; do
TRI_GRAPHS=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launch_rp$o.csv python tools/c2_profile.py --steps 3 --c3 --opt rerank_pairs_minkp=$o > gpurun_out/c3_ncu.log 2>&1
done
