mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --scores iid > gpurun_out/bench_iid.log 2>&1
cat gpurun_out/pytest_gpu.log; python -c "
import json
for f in ('gpurun_out/bench.log','gpurun_out/bench_iid.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f, round(d['value']), round(d['ms_per_step'],3), {k:round(r[k],3) for k in ('select_ms','attn_fwd_ms','attn_bwd_ms','frac','step_frac')})
"
mkdir -p gpurun_out; rm -f gpurun_out/time_fwd.log
for v in pp6 pp4; do SKB_LIB_PATH=paper_2406_16747_b200/_build/$v/libsparsek_b200.so timeout 300 python tools/time_fwd.py recency >> gpurun_out/time_fwd.log 2>&1; done
timeout 300 python tools/time_fwd.py recency >> gpurun_out/time_fwd.log 2>&1
cat gpurun_out/time_fwd.log
