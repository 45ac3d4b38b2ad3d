timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py 2 > gpurun_out/launches.log 2>&1
python tools/launch_table.py gpurun_out/launches.csv | grep skb
for sc in recency iid; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --scores $sc > gpurun_out/bench_$sc.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/bench_$sc.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$sc', round(d['value']), round(d['ms_per_step'],3), {k:round(r[k],3) for k in ('select_ms','attn_fwd_ms','attn_bwd_ms','frac','step_frac')})
"; done
