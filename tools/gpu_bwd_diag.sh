# selected-pass timeline (trace build) + source-level ncu of the backward kernels and the forward
mkdir -p gpurun_out
SKB_LIB_PATH=$PWD/paper_2406_16747_b200/_trsel/libsparsek_b200.so timeout 300 python tools/trace_selp.py > gpurun_out/trace_selp.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_dkdv_sel_tc|k_bwd_dq_p|k_fwd_p" -s 3 -c 3 -o gpurun_out/prof_bwd python tools/profile_step.py 2 > gpurun_out/ncu_bwd.log 2>&1
tail -3 gpurun_out/ncu_bwd.log
