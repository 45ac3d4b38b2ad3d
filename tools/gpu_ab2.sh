bash tools/gpu_ab.sh
SKB_LIB_PATH=paper_2406_16747_b200/_trace/libsparsek_b200.so timeout 300 python tools/trace_win.py | sed -n 9,13p
