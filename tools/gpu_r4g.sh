#!/bin/bash
# per-class table in shared memory (STK_MU_SMEM=1) against the default stream kernel; full suite + bench of the default
mkdir -p gpurun_out
T=${1:-r4g}
STK_EXTRA_FLAGS="-DSTK_MU_SMEM=1" python paper_1604_07994_b200/build.py --force > /dev/null 2>> gpurun_out/$T.build.err
timeout 240 python tools/time_ops.py cfg3 256 mu_smem >> gpurun_out/$T.ops.log 2>&1
timeout 240 python tools/time_ops.py cols 256 mu_smem >> gpurun_out/$T.ops.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/$T.parity_mu_smem.log 2>&1; echo "exit $?" >> gpurun_out/$T.parity_mu_smem.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/$T.bench_mu_smem.json 2> gpurun_out/$T.bench_mu_smem.err
python paper_1604_07994_b200/build.py --force > /dev/null 2>> gpurun_out/$T.build.err
timeout 240 python tools/time_ops.py cfg3 256 default >> gpurun_out/$T.ops.log 2>&1
timeout 240 python tools/time_ops.py cols 256 default >> gpurun_out/$T.ops.log 2>&1
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$T.bench_ref.json 2> gpurun_out/$T.bench_ref.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T.smoke.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/$T.gputest.log 2>&1; echo "exit $?" >> gpurun_out/$T.gputest.log
