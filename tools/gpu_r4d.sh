#!/bin/bash
# ncu --set full of the level-0 stream kernels at cfg3 n=256 with warp-state (stall) metrics
mkdir -p gpurun_out
T=${1:-r4d}
python paper_1604_07994_b200/build.py > /dev/null
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:k_stream -c 7 -o gpurun_out/$T.apply python tools/prof_apply.py cfg3 256 > gpurun_out/$T.ncu.log 2>&1
ncu -i gpurun_out/$T.apply.ncu-rep --page raw --csv > gpurun_out/$T.apply_raw.csv 2>/dev/null
