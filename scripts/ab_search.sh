# A/B device time of the search (one CUDA graph per search, L2 flushed) for builds of the
# library, interleaved over rounds (run under gpurun):
#   bash scripts/ab_search.sh "abtest/a.so abtest/b.so" [rounds] [domains...]
so=paper_2506_01099_b200/libbenelux_b200.so; cp $so /tmp/cur.so
libs=$1; rounds=${2:-3}; shift 2
for i in $(seq $rounds); do
  for v in $libs; do
    cp $v $so
    TAG=$v python scripts/time_search.py --reps 50 "$@" 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['tag'], d['hi'], 'median', round(d['median_ms'],4), 'min', round(d['min_ms'],4), d['kernels_ms'], 'surv', d['survivors'], 'cand', d['candidates'])"
  done
done
cp /tmp/cur.so $so
