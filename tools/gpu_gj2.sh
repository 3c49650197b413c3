timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q -k "switch or solve_matches" > gpurun_out/gj2.pytest.log 2>&1; echo "exit $?" >> gpurun_out/gj2.pytest.log
for v in 0 1; do echo "== STK_GJ_GRID=$v"; STK_GJ_GRID=$v timeout 200 python tools/time_assemble.py 2>&1 | tail -3; done > gpurun_out/gj2.log 2>&1
