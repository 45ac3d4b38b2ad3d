mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_tc" -s 1 -c 1 -o gpurun_out/prof_fwd python tools/profile_step.py 2 > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/ncu_full.log
