mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_gpu.py -q -x 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_decode.csv python tools/profile_decode.py 3 8192 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_decode.csv
timeout 600 python bench.py --workload decode --steps 20 --warmup 5 > gpurun_out/bench_decode.log 2>&1; cut -c1-400 gpurun_out/bench_decode.log
