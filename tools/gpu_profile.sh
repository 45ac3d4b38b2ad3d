# Round evidence: launch list of the bench command, one ncu --set full capture of each attention kernel.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py 2 > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_p|k_bwd_prep|k_bwd_dkdv_sel_tc|k_bwd_dkdv_win_tc|k_bwd_dq_p|k_rank_before|k_rank_after_warp|k_tau_chunks" -s 10 -c 10 -o gpurun_out/prof_attn python tools/profile_step.py 3 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/prof_attn.ncu-rep
