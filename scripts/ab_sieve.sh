# A/B of the exact sieve between builds of the library (run under gpurun):
#   bash scripts/ab_sieve.sh "abtest/old.so abtest/new.so" [rounds]
# prints one JSON line per build and round (scripts/sieve_variants.py child: timing + hashes)
so=paper_2506_01099_b200/libbenelux_b200.so; cp $so /tmp/cur.so
for i in $(seq ${2:-2}); do
  for v in $1; do
    cp $v $so
    echo "$v $(python scripts/sieve_variants.py child 2>&1 | tail -1)"
  done
done
cp /tmp/cur.so $so
