# quick loop: backward/forward parity tests + per-kernel launch times of the bench step
# usage: bash tools/gpu_quick.sh [pytest -k expr] [tag]
mkdir -p gpurun_out
K=${1:-"core or parity_configs or chunked"}
T=${2:-q}
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/t_$T.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_$T.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$T.csv python tools/profile_step.py 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/l_$T.csv | grep skb | grep -v "mean_us=      [0-9]\.[0-9]"
