for v in 16 32; do echo "== STK_GW_N=$v"; STK_GW_N=$v timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | grep "level 2\|without\|row_n=16"; done > gpurun_out/gw.log 2>&1
