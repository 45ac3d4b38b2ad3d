# compute-sanitizer memcheck over the kernels added late in round 2: the
# unified key-major backward (64-query tiles, default; and the 96/128-query
# opt-in), the CTA-pair selected pass, the decode control (a CTA per sequence,
# stream arrays staged in shared memory) and combine, with capped grids so
# every ring wraps (SKB_MAX_CTAS).
mkdir -p gpurun_out
run() {
  name=$1; shift
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 "$@" > gpurun_out/san_r2b_$name.log 2>&1
  echo "$name rc=$?"; grep -E "ERROR SUMMARY|passed|failed|^ok|^BAD" gpurun_out/san_r2b_$name.log | tail -3
}
SKB_MAX_CTAS=3 run unified python tests/scripts/persist_check.py
SKB_MAX_CTAS=3 SKB_BWD_QTILE=96 run kmaj96 python tests/scripts/persist_check.py
SKB_MAX_CTAS=4 SKB_BWD_UNI=0 SKB_BWD_PAIR=1 run pair python tests/scripts/persist_check.py small
run decode python -m pytest tests/test_decode_gpu.py tests/test_snapshot_gpu.py -q -x
run linmixdec python -m pytest tests/test_linmix_gpu.py -q -x -k decode
