#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x -k "apply or tiled or classification or smoother" > gpurun_out/d15.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/d15.pytest.log
for w in "cfg2 128" "cfg3 256" "cfg4 512"; do
  timeout 300 python tools/time_kernels.py $w 1 nosolve >> gpurun_out/d15.time.log 2>&1
done
timeout 300 python tools/prof_levels.py cfg2 128 > gpurun_out/d15.levels.log 2>&1
