#!/bin/bash
# cluster-fused coarse V-cycle: parity + timing; ncu full of the pressure passes
mkdir -p gpurun_out
T=${1:-r3a}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "coarse_level_kernel_paths or uzawa" > gpurun_out/$T.paths.log 2>&1; echo "exit $?" >> gpurun_out/$T.paths.log
timeout 400 python tools/prof_levels.py cfg3 256 > gpurun_out/$T.levels.log 2>&1
STK_FUSED_GRID=1 timeout 400 python tools/prof_levels.py cfg3 256 > gpurun_out/$T.levels_grid.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"k_stream<0, (3|4)>" -c 4 -o gpurun_out/$T.pp python tools/step_profiled.py cfg3 > gpurun_out/$T.ncu_pp.log 2>&1
