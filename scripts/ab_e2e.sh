# A/B of the public-API wall (scripts/time_e2e.py) for builds of the library (under gpurun)
so=paper_2506_01099_b200/libbenelux_b200.so; cp $so /tmp/cur.so
for i in $(seq ${2:-3}); do for v in $1; do cp $v $so; TAG=$v python scripts/time_e2e.py; done; done
cp /tmp/cur.so $so
