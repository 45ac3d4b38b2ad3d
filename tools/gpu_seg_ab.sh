mkdir -p gpurun_out
for scores in iid recency; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tau" --csv --log-file gpurun_out/seg.csv python tools/profile_step.py 2 $scores > /dev/null 2>&1
  echo "$scores: $(python tools/launch_table.py gpurun_out/seg.csv | awk '{print $1, $NF}' | tr '\n' ' ')"
done
timeout 600 python -m pytest tests -m gpu -x -q -k "select or tau or core or stream" 2>&1 | tail -1
timeout 400 python bench.py --scores iid --no-e2e --no-secondary --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('iid', l['ms_per_step'], l['roofline']['select_ms'])"
