#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x -k "apply or tiled or classification or smoother" > gpurun_out/d8.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/d8.pytest.log
for w in "cfg2 128" "cfg3 256" "cfg4 512"; do
  timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d8.time.log 2>&1
done
STK_KCHUNK=16 timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d8.time.log 2>&1
STK_KCHUNK=32 timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d8.time.log 2>&1
STK_KCHUNK=16 timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d8.time.log 2>&1
STK_KCHUNK=4 timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d8.time.log 2>&1
