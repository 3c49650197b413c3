#!/bin/bash
# per-level V-cycle profile at cfg3 n=256, form comparison (a4), ncu of the level-0 kernels
mkdir -p gpurun_out
T=${1:-r2k}
python paper_1604_07994_b200/build.py > /dev/null
timeout 600 python tools/prof_levels.py cfg3 256 > gpurun_out/$T.levels.log 2>&1
timeout 900 python tools/form_compare.py 128 > gpurun_out/$T.forms.json 2> gpurun_out/$T.forms.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream|k_listx" -c 6 \
   -o gpurun_out/$T.full python tools/prof_apply.py cfg3 256 > gpurun_out/$T.ncu.log 2>&1
