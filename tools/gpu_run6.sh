mkdir -p gpurun_out; rm -f gpurun_out/time_fwd.log
timeout 300 python tools/time_fwd.py recency >> gpurun_out/time_fwd.log 2>&1
timeout 300 python tools/time_fwd.py iid >> gpurun_out/time_fwd.log 2>&1
SKB_LIB_PATH=paper_2406_16747_b200/_build/tr/libsparsek_b200.so timeout 300 python tools/trace_fwd.py recency > gpurun_out/trace.log 2>&1
timeout 600 python -m pytest tests/test_core_gpu.py -q -x 2>&1 | tail -5 > gpurun_out/pytest_core.log
cat gpurun_out/time_fwd.log gpurun_out/trace.log gpurun_out/pytest_core.log
