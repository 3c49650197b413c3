#!/bin/bash
# decoupled-warp stream kernel (STK_DECOUPLE): level-0 op times for variants, parity of the variant, P1-P0 solve fix
mkdir -p gpurun_out
T=${1:-r4b}
run_variant() {
  lab=$1; fl=$2
  STK_EXTRA_FLAGS="$fl" python paper_1604_07994_b200/build.py --force > /dev/null 2>> gpurun_out/$T.build.err
  timeout 240 python tools/time_ops.py cfg3 256 $lab >> gpurun_out/$T.ops.log 2>&1 || echo "$lab cfg3 FAILED/timeout $?" >> gpurun_out/$T.ops.log
}
run_variant default ""
run_variant dec3 "-DSTK_DECOUPLE=1"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/$T.parity_dec3.log 2>&1; echo "exit $?" >> gpurun_out/$T.parity_dec3.log
timeout 240 python tools/time_ops.py cols 256 dec3 >> gpurun_out/$T.ops.log 2>&1
run_variant dec6 "-DSTK_DECOUPLE=1 -DSTK_PREF=6"
run_variant dec4 "-DSTK_DECOUPLE=1 -DSTK_PREF=4"
run_variant dec3_r128 "-DSTK_DECOUPLE=1 -DSTK_REGS_AR=128"
run_variant dec6_r128 "-DSTK_DECOUPLE=1 -DSTK_PREF=6 -DSTK_REGS_AR=128"
run_variant pref6 "-DSTK_PREF=6"
python paper_1604_07994_b200/build.py --force > /dev/null
timeout 900 python -m pytest tests/test_gpu_p1p0.py -q > gpurun_out/$T.p0.log 2>&1; echo "exit $?" >> gpurun_out/$T.p0.log
