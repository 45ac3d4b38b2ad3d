# A/B: parity tests, bench with an env toggle (AB_VAR) off/on, launch table; summary printed last.
V=${AB_VAR:-SKB_DQ_PERSIST}
mkdir -p gpurun_out
T=$(python -m pytest tests/test_core_gpu.py tests/test_chunked_gpu.py tests/test_api_gpu.py -x -q 2>&1 | tail -1)
R=""
for v in 0 1; do
  R="$R
$(env $V=$v python bench.py --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$V=$v', 'ms/step', round(d['ms_per_step'],3), 'sel', round(r['select_ms'],3), 'fwd', round(r['attn_fwd_ms'],3), 'bwd', round(r['attn_bwd_ms'],3))")"
done
ncu --metrics gpu__time_duration.sum --clock-control none -s 1 -c 40 --csv --log-file gpurun_out/ab_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > /dev/null 2>&1
python tools/launch_table.py gpurun_out/ab_launches.csv 2>&1 | grep "skb::" | grep -v "k_fill\|k_to_float\|k_tau_overflow\|k_tau_chunks_big\|k_union\|k_ever\|k_sel_items\|k_jvp\|k_tau_mono"
echo "TESTS: $T"
echo "$R"
