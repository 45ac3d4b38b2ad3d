# A/B of several alternative library builds (args) against the in-tree one: bench phases, twice each, interleaved
for rep in 1 2; do
  for L in paper_2406_16747_b200/libsparsek_b200.so "$@"; do
    SKB_LIB_PATH=$PWD/$L timeout 200 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$L', 'ms/step', round(d['ms_per_step'],3), 'sel', round(r['select_ms'],3), 'fwd', round(r['attn_fwd_ms'],3), 'bwd', round(r['attn_bwd_ms'],3))"
  done
done
