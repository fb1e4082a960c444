# k_heavy_screen register budget: builds with __launch_bounds__(256, M) for M = 6, 7, 8 and
# the matching grid (BNX_HEAVY_GRID = M), 2^32 search (run under gpurun)
so=paper_2506_01099_b200/libbenelux_b200.so; cp $so /tmp/cur.so
for r in 1 2; do
  for m in 8 7 6; do
    cp abtest/lb$m.so $so
    BNX_HEAVY_GRID=$m TAG=lb$m timeout 60 python scripts/time_search.py --reps 50 1:4294967295 | cut -c1-200
  done
done
cp /tmp/cur.so $so
