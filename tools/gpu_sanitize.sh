# compute-sanitizer over the persistent kernels with 2 CTAs (many items per CTA, ring wrap-arounds)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  SKB_MAX_CTAS=2 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tests/scripts/persist_check.py small > gpurun_out/san2_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok |BAD" gpurun_out/san2_$tool.log | tail -4
done
