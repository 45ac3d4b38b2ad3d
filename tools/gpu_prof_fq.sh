mkdir -p gpurun_out
for v in 0 1; do
SKB_BWD_DQPASS=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_fq$v.csv python tools/profile_step.py 2 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_dkdv_sel_tc|k_bwd_dkdv_win_tc" -s 2 -c 2 -o gpurun_out/prof_fq python tools/profile_step.py 2 > gpurun_out/ncu_fq.log 2>&1
tail -2 gpurun_out/ncu_fq.log
