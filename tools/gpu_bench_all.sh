# Round-end style bench lines (default, iid, decode, reference arm) -> gpurun_out/bench_*.json
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_recency.json 2> gpurun_out/bench_recency.err
python bench.py --scores iid --no-cpu-baseline > gpurun_out/bench_iid.json 2> gpurun_out/bench_iid.err
python bench.py --workload decode --no-cpu-baseline > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for f in gpurun_out/bench_*.json; do echo "== $f"; tail -1 $f | cut -c1-400; done
