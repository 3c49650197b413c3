#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x -k "apply or tiled or classification or smoother" > gpurun_out/d5.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/d5.pytest.log
for w in "cfg2 128" "cfg3 256" "cfg4 512"; do
  timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d5.time.log 2>&1
  STK_SKIP_IRR=1 timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d5.time.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/d5.bench.json 2> gpurun_out/d5.bench.err
timeout 300 python tools/prof_apply.py cfg4 512 > gpurun_out/d5.plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 1 -c 1 -o gpurun_out/d5_apply512 python tools/prof_apply.py cfg4 512 > gpurun_out/d5.ncu.log 2>&1
