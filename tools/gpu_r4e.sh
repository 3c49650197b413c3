#!/bin/bash
# distributed TMA issue (STK_PROD4) and two rows per thread (STK_NR2_MASK): level-0 op times + parity
mkdir -p gpurun_out
T=${1:-r4e}
run_variant() {
  lab=$1; fl=$2
  STK_EXTRA_FLAGS="$fl" python paper_1604_07994_b200/build.py --force > /dev/null 2>> gpurun_out/$T.build.err
  timeout 240 python tools/time_ops.py cfg3 256 $lab >> gpurun_out/$T.ops.log 2>&1 || echo "$lab cfg3 FAILED/timeout $?" >> gpurun_out/$T.ops.log
}
run_variant prod4 ""
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/$T.parity_prod4.log 2>&1; echo "exit $?" >> gpurun_out/$T.parity_prod4.log
run_variant nr2_232 "-DSTK_NR2_MASK=31 -DSTK_REGS_NR2=232"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/$T.parity_nr2.log 2>&1; echo "exit $?" >> gpurun_out/$T.parity_nr2.log
timeout 240 python tools/time_ops.py cols 256 nr2_232 >> gpurun_out/$T.ops.log 2>&1
run_variant nr2_168 "-DSTK_NR2_MASK=31 -DSTK_REGS_NR2=168"
run_variant nr2_200 "-DSTK_NR2_MASK=31 -DSTK_REGS_NR2=200"
run_variant prod1 "-DSTK_PROD4=0"
python paper_1604_07994_b200/build.py --force > /dev/null
