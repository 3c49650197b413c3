python paper_1604_07994_b200/build.py > /dev/null
STK_FSWEEP=0 timeout 120 python tools/dbg_fsweep.py cfg1 64 > gpurun_out/r2p.log 2>&1
CUDA_LAUNCH_BLOCKING=1 STK_FSWEEP=1 timeout 120 python tools/dbg_fsweep.py cfg1 64 >> gpurun_out/r2p.log 2>&1
