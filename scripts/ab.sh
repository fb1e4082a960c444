# A/B device timing of builds of the library (run under gpurun):
#   bash scripts/ab.sh "abtest/old.so abtest/new.so ..." [rounds]
so=paper_2506_01099_b200/libbenelux_b200.so; cp $so /tmp/cur.so
for i in $(seq ${2:-3}); do
  for v in $1; do
    cp $v $so
    python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-sieve --no-2p40 2>/dev/null | python -c "
import json,sys; b=json.loads(sys.stdin.read()); print('$v', round(b['ms_per_step'],5))"
  done
done
cp /tmp/cur.so $so
