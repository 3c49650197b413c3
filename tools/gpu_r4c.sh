#!/bin/bash
# P1-P0 solve with the element-local pressure term; ncu --set full of the apply / vel kernels with warp-state (stall) metrics
mkdir -p gpurun_out
T=${1:-r4c}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_p1p0.py -q > gpurun_out/$T.p0.log 2>&1; echo "exit $?" >> gpurun_out/$T.p0.log
timeout 600 python tools/prof_apply.py cfg3 256 > gpurun_out/$T.prof_plain.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"k_stream<0, (0|2)>" -c 4 -o gpurun_out/$T.apply python tools/prof_apply.py cfg3 256 > gpurun_out/$T.ncu.log 2>&1
ncu -i gpurun_out/$T.apply.ncu-rep --page raw --csv > gpurun_out/$T.apply_raw.csv 2>/dev/null
