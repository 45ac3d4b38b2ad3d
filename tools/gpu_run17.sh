mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_tc|k_bwd_dkdv_tc|k_bwd_dq_tc" -s 4 -c 4 -o gpurun_out/prof_r1 python tools/profile_step.py 3 > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/ncu_full.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_torchrun.log 2>&1
tail -c 600 gpurun_out/bench_torchrun.log
