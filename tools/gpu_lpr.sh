for v in 0 4 8 16; do echo "== LPR $v"; STK_ROW_LPR=$v timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | tail -4; done > gpurun_out/lpr.log 2>&1
