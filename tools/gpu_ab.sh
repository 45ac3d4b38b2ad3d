# same-box A/B of the bench step's attention kernels: product library vs _exp$1 (twice, interleaved)
mkdir -p gpurun_out
V=${1:-2}
for rep in 1 2; do
for lib in $PWD/paper_2406_16747_b200/libsparsek_b200.so $PWD/paper_2406_16747_b200/_exp$V/libsparsek_b200.so; do
  tag=$(basename $(dirname $lib))
  SKB_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv python tools/profile_step.py 2 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/ab.csv | grep "k_fwd_p\|k_bwd_dkdv\|k_bwd_dq\|k_bwd_kmaj" | sed -e 's/(.*mean_us=/ /' -e 's/void skb::<unnamed>:://' -e 's/skb::<unnamed>:://' | sed "s/^/$tag r$rep /"
done
done
