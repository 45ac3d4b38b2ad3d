mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rank_leave|k_tau_chunks" -s 2 -c 2 -o gpurun_out/prof_sel python tools/profile_step.py 2 > gpurun_out/ncu_sel.log 2>&1
tail -2 gpurun_out/ncu_sel.log
