# unified pass query-tile A/B (same box) + parity subset on the default
mkdir -p gpurun_out
for rep in 1 2; do
for v in 0 96 128; do
  SKB_BWD_QTILE=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qt.csv python tools/profile_step.py 2 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/qt.csv | grep "kmaj\|dkdv_win_tc<128, 0, 1>" | sed "s/^/QTILE=$v r$rep /" | cut -c1-40,71-
done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "${1:-core or parity_configs or chunked or api}" 2>&1 | tail -2
