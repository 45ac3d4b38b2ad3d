# selected pass A/B: product vs _exp2 build, pair on/off; then correctness on the product build
mkdir -p gpurun_out
for v in "" 2; do
  lib=$PWD/paper_2406_16747_b200/libsparsek_b200.so
  [ -n "$v" ] && lib=$PWD/paper_2406_16747_b200/_exp$v/libsparsek_b200.so
  SKB_BWD_PAIR=0 SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bwd_dkdv --csv --log-file gpurun_out/ab_$v.csv python tools/profile_step.py 2 > /dev/null 2>&1
  grep -h k_bwd_dkdv gpurun_out/ab_$v.csv | awk -F'","' -v v="lib$v" '{print v, substr($5,1,40), $NF}'
done
SKB_BWD_PAIR=0 SKB_LIB_PATH=$PWD/paper_2406_16747_b200/_trsel/libsparsek_b200.so timeout 300 python tools/trace_selp.py > gpurun_out/trace_il.txt 2>&1; grep -A12 "CTA 100" gpurun_out/trace_il.txt
SKB_BWD_PAIR=0 timeout 900 python -m pytest tests -m gpu -x -q -k "core or parity_configs or chunked" 2>&1 | tail -2
