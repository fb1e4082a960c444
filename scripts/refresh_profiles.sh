# Everything profiles/ holds, in one GPU call (run under gpurun; summaries are made here after):
#   bench line, launch lists at 2^32 and 2^40, ncu --set full of the heavy kernels, the
#   paper range, beyond the paper, shard balance.
set -x
mkdir -p gpurun_out/refresh
O=gpurun_out/refresh
python bench.py > $O/bench.json 2> $O/bench.err || exit 1
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/gen32.csv python scripts/profile_search.py 32 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/gen40.csv python scripts/profile_search.py 40 3 > /dev/null 2>&1
for k in k_heavy_screen k_heavy_exact k_tail k_tail_heavy; do
  ncu --set full --import-source on --clock-control none -k $k -s 1 -c 1 -o $O/full_$k -f \
      python scripts/profile_search.py 32 > $O/ncu_$k.log 2>&1
done
ncu --set full --import-source on --clock-control none -k k_heavy_sieve -s 1 -c 1 -o $O/full_2p40_k_heavy_sieve -f \
    python scripts/profile_search.py 40 3 > $O/ncu_sieve.log 2>&1
python scripts/paper_range.py > $O/paper_range.jsonl 2> $O/paper_range.err
python scripts/beyond_paper.py 1400000000000 2^44 2^45 2^46 2^47 2^48 > $O/beyond_paper.jsonl 2> $O/beyond.err
{ python scripts/shard_balance.py 2^40 8; python scripts/shard_balance.py 2^44 8; } > $O/shard_balance.jsonl 2> $O/shard.err
ls -la $O
