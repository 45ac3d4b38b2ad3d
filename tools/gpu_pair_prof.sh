mkdir -p gpurun_out
for v in 0 1; do
SKB_BWD_PAIR=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_dkdv_sel" -s 1 -c 1 -o gpurun_out/prof_pair$v python tools/profile_step.py 2 > gpurun_out/ncu_pair$v.log 2>&1
tail -1 gpurun_out/ncu_pair$v.log
done
