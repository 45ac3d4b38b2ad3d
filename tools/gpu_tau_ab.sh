# tau band-sort radix width A/B: select kernels of the bench step, product (4 bits) vs _exp5/6/8
mkdir -p gpurun_out
for rep in 1 2; do
for v in "" 5 6; do
  lib=$PWD/paper_2406_16747_b200/libsparsek_b200.so
  [ -n "$v" ] && lib=$PWD/paper_2406_16747_b200/_exp$v/libsparsek_b200.so
  SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tau_chunks|k_tau_seg" --csv --log-file gpurun_out/tau.csv python tools/profile_step.py 2 iid > /dev/null 2>&1
  SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tau_chunks" --csv --log-file gpurun_out/tau2.csv python tools/profile_step.py 2 > /dev/null 2>&1
  echo "bits=${v:-4} r$rep iid: $(python tools/launch_table.py gpurun_out/tau.csv | awk '{print $NF}' | tr '\n' ' ') recency: $(python tools/launch_table.py gpurun_out/tau2.csv | awk '{print $NF}' | tr '\n' ' ')"
done
done
SKB_LIB_PATH=$PWD/paper_2406_16747_b200/_exp6/libsparsek_b200.so timeout 600 python -m pytest tests -m gpu -x -q -k "select or tau or core" 2>&1 | tail -1
