#!/bin/bash
# round-2 first GPU check: R15 coarse coefficients, integer parity, solves on tiled levels,
# convergence at BASELINE sizes with GMRES(30) + V-cycle
mkdir -p gpurun_out
T=${1:-r2a}
python paper_1604_07994_b200/build.py > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/$T.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T.pytest.log
for c in "cfg3 64 30" "cfg3 128 30" "cfg3 256 30" "cfg5 64 30" "cfg5 128 30" "cfg5 256 30" "cfg4 128 30" "cfg4 256 30" "cfg2 128 0" "cfg1 64 0"; do
  timeout 300 python tools/solve_probe.py $c >> gpurun_out/$T.probe.log 2>&1
done
