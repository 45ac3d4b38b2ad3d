mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$1.csv python tools/profile_step.py 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/l_$1.csv | grep "k_fwd_p\|k_bwd"
timeout 900 python -m pytest tests -m gpu -x -q -k "core or parity_configs or chunked" 2>&1 | tail -1
