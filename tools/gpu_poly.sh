mkdir -p gpurun_out
for rep in 1 2; do
for v in "" 1 5 3; do
  lib=$PWD/paper_2406_16747_b200/libsparsek_b200.so
  [ -n "$v" ] && lib=$PWD/paper_2406_16747_b200/_exp$v/libsparsek_b200.so
  SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fwd_p --csv --log-file gpurun_out/poly.csv python tools/profile_step.py 2 > /dev/null 2>&1
  echo "mask=${v:-0} r$rep $(python tools/launch_table.py gpurun_out/poly.csv | awk '{print $NF}')"
done
done
