mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 1 -c 60 --csv --log-file gpurun_out/iid_launches.csv python bench.py --scores iid --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/iid_launches.csv 2>&1 | grep "skb::"
