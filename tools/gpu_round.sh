# Round evidence in one call: GPU tests, launch list + ncu captures, bench lines.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 bash tools/gpu_profile.sh > gpurun_out/profile.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 400 python bench.py --workload decode > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 400 python bench.py --scores iid --no-secondary --no-cpu-baseline > gpurun_out/bench_iid.json 2> gpurun_out/bench_iid.err
tail -2 gpurun_out/gputest.log
