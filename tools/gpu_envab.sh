# same-box A/B of an env knob: bash tools/gpu_envab.sh VAR VALUE_A VALUE_B [pytest -k expr]
mkdir -p gpurun_out
V=$1; A=$2; B=$3; K=${4:-}
for rep in 1 2; do
for val in $A $B; do
  env $V=$val timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/envab.csv python tools/profile_step.py 2 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/envab.csv | grep "k_fwd_p\|k_bwd_dkdv\|k_bwd_dq\|k_bwd_kmaj" | sed "s/^/$V=$val r$rep /" | cut -c1-45,71-
done
done
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -2; fi
