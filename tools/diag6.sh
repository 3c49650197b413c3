#!/bin/bash
for w in "cfg2 128" "cfg4 512"; do
  timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d6.time.log 2>&1
  STK_SKIP_IRR=1 timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d6.time.log 2>&1
done
timeout 300 python tools/prof_apply.py cfg2 128 > gpurun_out/d6.plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_list|k_stream" -s 2 -c 2 -o gpurun_out/d6_list128 python tools/prof_apply.py cfg2 128 > gpurun_out/d6.ncu.log 2>&1
