#!/bin/bash
# stream-kernel variants: unroll mask, register caps (level-0 op times at cfg3 n=256)
mkdir -p gpurun_out
T=${1:-r3d}
for v in "default|" "unroll_all|-DSTK_UNROLL3_MASK=31" "unroll_apply|-DSTK_UNROLL3_MASK=5" "regsP96|-DSTK_REGS_P=96" "regsP64|-DSTK_REGS_P=64" "regsAR128|-DSTK_REGS_AR=128" "regsAR104|-DSTK_REGS_AR=104"; do
  lab=${v%%|*}; fl=${v#*|}
  STK_EXTRA_FLAGS="$fl" python paper_1604_07994_b200/build.py --force > /dev/null 2>> gpurun_out/$T.build.err
  timeout 300 python tools/time_ops.py cfg3 256 $lab >> gpurun_out/$T.ops.log 2>&1
  timeout 300 python tools/time_ops.py cols 256 $lab >> gpurun_out/$T.ops.log 2>&1
done
python paper_1604_07994_b200/build.py --force > /dev/null
