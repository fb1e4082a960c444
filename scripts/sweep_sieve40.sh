# k_heavy_sieve CTA size x chunk length x CTAs per SM at 2^40 and 1.4e12 (run under gpurun)
for cfg in "256 768 40" "128 384 40" "128 384 80" "128 768 80" "64 256 120" "128 256 80" "256 768 40"; do
  set -- $cfg
  BNX_SIEVE_THREADS=$1 BNX_HEAVY_KC=$2 BNX_SIEVE_GRID=$3 timeout 120 python scripts/time_search.py --reps 20 1:1099511627775 1:1400000000000 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('threads $1 kc $2 grid $3', d['hi'], 'median', round(d['median_ms'],4), d['kernels_ms']['screen'])"
done
