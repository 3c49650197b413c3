python paper_1604_07994_b200/build.py > /dev/null
for c in "cfg1 64" "cfg2 64" "cfg3 128" "cfg5 128"; do STK_FSWEEP=1 timeout 60 python tools/dbg_fsweep.py $c 2>&1 | grep -v "^  File\|^    \|Traceback" | head -3 >> gpurun_out/r2q7.log; done
