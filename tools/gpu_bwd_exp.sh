# selected-pass decomposition: product vs experiment builds (SKB_BWD_EXP=1/2/3), and the tau phase clocks
mkdir -p gpurun_out
for v in "" 1 2 3; do
  lib=$PWD/paper_2406_16747_b200/libsparsek_b200.so
  [ -n "$v" ] && lib=$PWD/paper_2406_16747_b200/_exp$v/libsparsek_b200.so
  SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bwd_dkdv_sel --csv --log-file gpurun_out/exp_sel$v.csv python tools/profile_step.py 2 > /dev/null 2>&1
done
SKB_LIB_PATH=$PWD/paper_2406_16747_b200/_trace/libsparsek_b200.so timeout 300 python tools/trace_tau.py > gpurun_out/trace_tau.txt 2>&1
SKB_LIB_PATH=$PWD/paper_2406_16747_b200/_trace/libsparsek_b200.so timeout 300 python tools/trace_tau.py iid >> gpurun_out/trace_tau.txt 2>&1
for v in "" 1 2 3; do grep -h k_bwd_dkdv_sel gpurun_out/exp_sel$v.csv | awk -F'","' -v v="exp$v" '{print v, $NF}'; done
cat gpurun_out/trace_tau.txt
