#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2r}
python paper_1604_07994_b200/build.py > /dev/null
for c in "cfg1 64" "cfg2 64" "cfg3 128" "cfg5 128"; do STK_FSWEEP=1 timeout 60 python tools/dbg_fsweep.py $c 2>&1 | grep -v "^  File\|^    \|Traceback" | head -3 >> gpurun_out/$T.dbg.log; done
timeout 300 python tools/prof_levels.py cfg3 256 > gpurun_out/$T.levels.log 2>&1
STK_FSWEEP=0 timeout 300 python tools/prof_levels.py cfg3 256 > gpurun_out/$T.levels0.log 2>&1
