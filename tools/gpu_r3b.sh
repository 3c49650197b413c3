#!/bin/bash
# P1-P0 apply parity; listx/free-slip regression; ncu pressure passes
mkdir -p gpurun_out
T=${1:-r3b}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_p1p0.py -q > gpurun_out/$T.p0.log 2>&1; echo "exit $?" >> gpurun_out/$T.p0.log
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled \
  -k regex:"k_stream<0, (3|4)>" -c 4 -o gpurun_out/$T.pp python tools/step_profiled.py cfg3 > gpurun_out/$T.ncu_pp.log 2>&1
