# ncu launch list of one 2^32 search + one --set full capture per heavy-path kernel (run under gpurun)
set -x
mkdir -p gpurun_out
python scripts/profile_search.py 32 > gpurun_out/ps.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/gen.csv python scripts/profile_search.py 32 > /dev/null 2>&1
for k in k_heavy_screen k_heavy_exact k_tail k_tail_heavy; do
ncu --set full --import-source on --clock-control none -k $k -s 1 -c 1 -o gpurun_out/full_$k -f python scripts/profile_search.py 32 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
