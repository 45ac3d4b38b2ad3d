for v in "" 1; do
  lib=$PWD/paper_2406_16747_b200/libsparsek_b200.so
  [ -n "$v" ] && lib=$PWD/paper_2406_16747_b200/_exp$v/libsparsek_b200.so
  for p in 0 1; do
  SKB_BWD_PAIR=$p SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bwd_dkdv_sel --csv --log-file gpurun_out/e1_$v$p.csv python tools/profile_step.py 2 > /dev/null 2>&1
  grep -h k_bwd_dkdv_sel gpurun_out/e1_$v$p.csv | awk -F'","' -v v="exp$v pair$p" '{print v, $NF}'
  done
done
