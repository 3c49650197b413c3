#!/bin/bash
# probe + timing + parity after the stream-kernel rewrite
timeout 60 ./tools/probe_tma_neg > gpurun_out/d2.probe.log 2>&1; echo "exit $?" >> gpurun_out/d2.probe.log
for kc in 8 16; do
  STK_KCHUNK=$kc timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d2.time.log 2>&1
done
STK_SKIP_IRR=1 timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d2.time.log 2>&1
timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d2.time.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity.py::test_solve_matches_direct_solution > gpurun_out/d2.pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/d2.pytest.log
