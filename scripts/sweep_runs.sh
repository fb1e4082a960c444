# Sweep of the screen's run partition and grid at 2^32 and 2^40 (run under gpurun): static
# share (BNX_HEAVY_RUN_FIRST /256), dynamic runs per CTA (BNX_HEAVY_RUNS), CTAs per SM
# (BNX_HEAVY_GRID); mean device time of one search over 100 repetitions.
for g in 7 6 8; do for r in 2 0 1 3 4 6; do for f in 128 64 192 224; do
  BNX_HEAVY_GRID=$g BNX_HEAVY_RUNS=$r BNX_HEAVY_RUN_FIRST=$f TAG="g$g r$r f$f" timeout 120 python scripts/time_search.py --reps 100 "$@" 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['tag'], d['hi'], 'mean', round(d['mean_ms'],4), 'median', round(d['median_ms'],4), d['kernels_ms']['screen'])"
done; done; done
