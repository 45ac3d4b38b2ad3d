rm -f gpurun_out/time_fwd.log
SKB_LIB_PATH=paper_2406_16747_b200/_build/e9/libsparsek_b200.so timeout 300 python tools/time_fwd.py recency
timeout 300 python tools/time_fwd.py recency
SKB_LIB_PATH=paper_2406_16747_b200/_build/e9/libsparsek_b200.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e9 bench', d['ms_per_step'], d['roofline']['attn_bwd_ms'])"
