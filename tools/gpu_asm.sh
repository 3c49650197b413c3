for v in 0 1; do echo "== STK_GJ_GRID=$v"; STK_GJ_GRID=$v timeout 200 python tools/time_assemble.py 2>&1 | tail -3; done > gpurun_out/asm.log 2>&1
