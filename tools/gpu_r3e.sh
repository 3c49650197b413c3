#!/bin/bash
# NEXT-3 1-GPU rung (weak ladder: n = 512 per GPU cube), P1-P0 GPU tests (fluxes)
mkdir -p gpurun_out
T=${1:-r3e}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_p1p0.py -q > gpurun_out/$T.p0.log 2>&1; echo "exit $?" >> gpurun_out/$T.p0.log
timeout 900 python bench.py --scaling weak --workload cols --steps 3 --no-cpu-baseline > gpurun_out/$T.weak_cols.json 2> gpurun_out/$T.weak_cols.err
timeout 1200 python bench.py --scaling weak --workload cfg4 --n 256 --steps 2 --no-cpu-baseline > gpurun_out/$T.weak_cfg4_256.json 2> gpurun_out/$T.weak_cfg4_256.err
