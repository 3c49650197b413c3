python paper_1604_07994_b200/build.py > /dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fsweep" -c 1 -o gpurun_out/r2s.fs python tools/prof_apply.py cfg3 256 > gpurun_out/r2s.ncu.log 2>&1
