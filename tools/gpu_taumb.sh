mkdir -p gpurun_out
for rep in 1 2; do
for v in "" 6 8; do
  lib=$PWD/paper_2406_16747_b200/libsparsek_b200.so
  [ -n "$v" ] && lib=$PWD/paper_2406_16747_b200/_exp$v/libsparsek_b200.so
  SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tau_chunks" --csv --log-file gpurun_out/tmb.csv python tools/profile_step.py 2 > /dev/null 2>&1
  echo "minb=${v:-4} r$rep $(python tools/launch_table.py gpurun_out/tmb.csv | awk '{print $NF}' | tr '\n' ' ')"
done
done
