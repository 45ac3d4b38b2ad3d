mkdir -p gpurun_out; rm -f gpurun_out/time_fwd.log
for v in e1 e2 e3; do SKB_LIB_PATH=paper_2406_16747_b200/_build/$v/libsparsek_b200.so timeout 300 python tools/time_fwd.py recency >> gpurun_out/time_fwd.log 2>&1; done
timeout 300 python tools/time_fwd.py recency >> gpurun_out/time_fwd.log 2>&1
cat gpurun_out/time_fwd.log
