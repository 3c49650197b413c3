#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x -k "apply or tiled or classification or smoother" > gpurun_out/d7.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/d7.pytest.log
for w in "cfg2 128" "cfg3 256" "cfg4 512"; do
  timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d7.time.log 2>&1
  STK_LIST_FORK=1 timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d7.time.log 2>&1
done
timeout 300 python tools/prof_apply.py cfg2 128 > gpurun_out/d7.plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_list|k_stream" --csv --log-file gpurun_out/d7.launches.csv python tools/prof_apply.py cfg2 128 > gpurun_out/d7.ncu.log 2>&1
