#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/d9.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/d9.pytest.log
for w in "cfg2 128" "cfg3 256" "cfg4 512"; do
  timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d9.time.log 2>&1
done
STK_SKIP_IRR=1 timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d9.time.log 2>&1
STK_KCHUNK=32 timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d9.time.log 2>&1
STK_KCHUNK=16 timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d9.time.log 2>&1
STK_LIST_FORK=1 timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d9.time.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/d9.bench.json 2> gpurun_out/d9.bench.err
