#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2n}
python paper_1604_07994_b200/build.py > /dev/null
timeout 300 python -m pytest tests/test_gpu_loopback.py -q > gpurun_out/$T.loop.log 2>&1; echo "exit $?" >> gpurun_out/$T.loop.log
timeout 600 python tools/solve_sweep.py cfg3 256 > gpurun_out/$T.sweep.log 2>&1
timeout 400 python tools/solve_sweep.py cfg5 256 >> gpurun_out/$T.sweep.log 2>&1
