# Round-2 evidence run on one B200 (under gpurun): GPU tests, bench lines (N=1, emulated
# N=2/4/8, the NCCL code path with one rank, the reference arm), and the ncu launch lists
# behind the roofline (profiles/).  Outputs in gpurun_out/r2_*.  Every step has its own timeout.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
for n in 2 4 8; do
  timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 --no-sieve --no-cpu-baseline > gpurun_out/r2_bench_gpus${n}_emulated.json 2> gpurun_out/r2_bench_gpus${n}_emulated.err; echo emul$n rc=$?
done
BNX_FORCE_DIST=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 --no-sieve --no-cpu-baseline > gpurun_out/r2_bench_force_dist.json 2> gpurun_out/r2_bench_force_dist.err; echo fdist rc=$?
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; echo ref rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_heavy_launches.csv python scripts/profile_search.py 32 > /dev/null 2>&1; echo ncu32 rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_heavy_launches_2p40.csv python scripts/profile_search.py 40 1 > /dev/null 2>&1; echo ncu40 rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sieve --no-2p40 > /dev/null 2>&1; echo ncubench rc=$?
timeout 600 python scripts/paper_range.py > gpurun_out/r2_paper_range.jsonl 2> gpurun_out/r2_paper_range.err; echo range rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k k_tail -c 1 -o gpurun_out/r2_k_tail python scripts/profile_search.py 32 > gpurun_out/r2_ncu_tail.log 2>&1; echo ncutail rc=$?
