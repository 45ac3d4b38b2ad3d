mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py 2 > gpurun_out/launches.log 2>&1
python tools/launch_table.py gpurun_out/launches.csv | grep skb
python -c "
import json
for f in ('gpurun_out/bench.log',):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f, round(d['value']), round(d['ms_per_step'],3), {k:round(r[k],3) for k in ('select_ms','attn_fwd_ms','attn_bwd_ms','frac','step_frac')})
"
SKB_LIB_PATH=paper_2406_16747_b200/_build/tr/libsparsek_b200.so timeout 300 python tools/trace_dq.py | sed -n 6,9p
