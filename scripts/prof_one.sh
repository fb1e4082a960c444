# One ncu --set full capture of kernel $1 in the second 2^${2:-32} search (run under gpurun)
mkdir -p gpurun_out
python scripts/profile_search.py ${2:-32} > gpurun_out/ps.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k $1 -s 1 -c 1 -o gpurun_out/full_$1 -f \
    python scripts/profile_search.py ${2:-32} > gpurun_out/ncu_$1.log 2>&1
