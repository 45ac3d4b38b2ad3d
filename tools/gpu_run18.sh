for v in 0 3; do SKB_FWD_VARIANT=$v timeout 300 python tools/time_fwd.py recency; SKB_FWD_VARIANT=$v timeout 300 python tools/time_fwd.py iid; done
SKB_FWD_VARIANT=3 timeout 600 python -m pytest tests/test_core_gpu.py -q -x 2>&1 | tail -3
