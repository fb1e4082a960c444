set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r2_pytest_gpu.txt
python bench.py --steps 10 --warmup 3 --no-extrapolation > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo bench rc=$?
python bench.py --gpus 2 --steps 5 --warmup 3 --no-sieve --no-cpu-baseline > gpurun_out/r2_bench_emul2.json 2> gpurun_out/r2_bench_emul2.err; echo emul rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo ref rc=$?
for o in 0 1 2 3; do BNX_HEAVY_ORDER=$o TAG=order$o python scripts/time_search.py 1:4294967295 1:1099511627775 1:1399999999999 ; done > gpurun_out/r2_order.jsonl 2>&1
cat gpurun_out/r2_order.jsonl
