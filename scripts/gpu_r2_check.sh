# round-2 scratch GPU check: targeted tests, cold-path trace, search timings, a short bench
set -x
python -m pytest tests/test_gpu_classes.py -x -q > gpurun_out/r2_pytest_cls.txt 2>&1; echo cls rc=$?
tail -15 gpurun_out/r2_pytest_cls.txt
BNX_TRACE=1 python -c "
import time, torch; torch.cuda.init(); torch.zeros(1).cuda()
import sys; sys.path.insert(0,'.')
from paper_2506_01099_b200 import _native
for S in (2**32, 1_400_000_000_000, 2**44, 2**48):
    c = _native.Context(0); t=time.perf_counter(); r=c.search(S, 3, None, 0); print('cold', S, len(r), (time.perf_counter()-t)*1e3, 'ms', flush=True); c.close()
" > gpurun_out/r2_trace.txt 2>&1
cat gpurun_out/r2_trace.txt
python scripts/time_search.py 1:4294967295 1:1099511627775 > gpurun_out/r2_time.jsonl 2>&1; cat gpurun_out/r2_time.jsonl
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r2_pytest_gpu.txt
