mkdir -p gpurun_out
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -q -x tests/test_decode_gpu.py 2>&1 | tail -40 > gpurun_out/pytest_decode.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_tc|k_bwd_dkdv_tc|k_bwd_dq_tc" -s 6 -c 4 -o gpurun_out/prof_attn python tools/profile_step.py 3 > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/*.log
