#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x -k "apply or tiled or classification or smoother" > gpurun_out/d3.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/d3.pytest.log
timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve > gpurun_out/d3.time.log 2>&1
STK_SKIP_IRR=1 timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d3.time.log 2>&1
timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d3.time.log 2>&1
STK_SKIP_IRR=1 timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d3.time.log 2>&1
STK_SKIP_IRR=1 timeout 300 python tools/prof_apply.py cfg4 512 > gpurun_out/d3.plain.log 2>&1 && \
STK_SKIP_IRR=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 1 -c 1 -o gpurun_out/d3_apply512 python tools/prof_apply.py cfg4 512 > gpurun_out/d3.ncu.log 2>&1
