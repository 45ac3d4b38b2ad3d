mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python tools/time_fwd.py recency > gpurun_out/time_fwd.log 2>&1
timeout 300 python tools/time_fwd.py iid >> gpurun_out/time_fwd.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_tc" -s 1 -c 1 -o gpurun_out/prof_fwd python tools/profile_step.py 2 > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/*.log
