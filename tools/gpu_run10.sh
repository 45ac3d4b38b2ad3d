mkdir -p gpurun_out
timeout 600 python bench.py --workload decode --steps 20 --warmup 5 > gpurun_out/bench_decode.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/bench_decode.log gpurun_out/bench.log
