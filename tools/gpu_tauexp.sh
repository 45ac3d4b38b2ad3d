for e in 0 1 2; do
  L=paper_2406_16747_b200/libsparsek_b200.so; [ $e != 0 ] && L=paper_2406_16747_b200/_trace/libx$e.so
  SKB_LIB_PATH=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tau" -c 6 --csv --log-file gpurun_out/tx$e.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "== exp $e"; python tools/launch_table.py gpurun_out/tx$e.csv | grep "k_tau_chunks("
done
