SKB_LIB_PATH=paper_2406_16747_b200/_build/tr/libsparsek_b200.so timeout 300 python tools/trace_bwd.py | head -12
