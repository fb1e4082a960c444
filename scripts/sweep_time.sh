# Median device time of whole searches (time_search.py, one graph per search, L2 flushed) per
# value of one environment knob (run under gpurun):
#   bash scripts/sweep_time.sh VAR "v1 v2 ..." domain [domain ...]
var=$1; vals=$2; shift 2
for v in $vals; do
  env $var=$v timeout 120 python scripts/time_search.py --reps 20 "$@" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$var=$v', d['hi'], 'median', round(d['median_ms'],4), d['kernels_ms'])"
done
