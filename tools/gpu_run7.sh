mkdir -p gpurun_out
SKB_LIB_PATH=paper_2406_16747_b200/_build/e8tr/libsparsek_b200.so timeout 300 python tools/trace_fwd.py recency > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
