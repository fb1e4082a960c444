# k_heavy_sieve mask mode at 2^32: kmin x sieve CTAs per SM (run under gpurun)
for g in 2 4 8; do
  for km in 0 32 128 512 2048; do
    if [ $km = 0 ]; then unset BNX_HEAVY_KMIN; else export BNX_HEAVY_KMIN=$km; fi
    BNX_SIEVE_GRID=$g timeout 60 python scripts/time_search.py --reps 30 1:4294967295 | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('grid $g kmin $km', round(d['median_ms'],4), d['kernels_ms'], d['survivors'], d['candidates'])"
  done
done
