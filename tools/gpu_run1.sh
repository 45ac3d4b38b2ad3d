set -x
mkdir -p gpurun_out
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --scores iid --no-cpu-baseline > gpurun_out/bench_iid.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py 2 > gpurun_out/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn -s 4 -c 4 -o gpurun_out/prof_attn python tools/profile_step.py 3 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/*.log
