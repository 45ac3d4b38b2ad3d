# compute-sanitizer memcheck over the round-2 kernels: K1 (tiled raw + staged
# Welford), the linear mix (fwd/bwd/decode), the CTA-pair projection GEMM with
# the streaming Welford, the opt-in fused-dQ backward, the decode head split.
mkdir -p gpurun_out
run() {
  name=$1; shift
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 "$@" > gpurun_out/san_r2_$name.log 2>&1
  echo "$name rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_r2_$name.log | tail -2
}
run score python -m pytest tests/test_score_gpu.py -q -x -k "257 or 130"
run linmix python -m pytest tests/test_linmix_gpu.py -q -x
run proj python -m pytest tests/test_proj_gpu.py -q -x -k "256-256 or 77"
SKB_BWD_FUSEDQ=1 run fusedq python tests/scripts/persist_check.py small
SKB_DEC_HS=16 SKB_DEC_FUSE=1 run decode python -m pytest tests/test_decode_gpu.py -q -x
