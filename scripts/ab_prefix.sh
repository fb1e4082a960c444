# Pipeline-prefix device time (BNX_STOP_AFTER = 1 count+scan, 2 + screen, 3 + exact, 0 all)
# for builds of the library (run under gpurun):  bash scripts/ab_prefix.sh "a.so b.so" [domain]
so=paper_2506_01099_b200/libbenelux_b200.so; cp $so /tmp/cur.so
for v in $1; do
  cp $v $so
  for s in 1 2 3 0; do
    BNX_STOP_AFTER=$s TAG="$v stop$s" python scripts/time_search.py --reps 50 ${2:-1:4294967295} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print(d['tag'], 'median', round(d['median_ms'],4), 'min', round(d['min_ms'],4))
    except Exception: print(l.strip())"
  done
done
cp /tmp/cur.so $so
