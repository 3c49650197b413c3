mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled or uzawa" > gpurun_out/rep.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/rep.pytest.log
for v in 1 0; do echo "== STK_VEL_REPEAT=$v"; STK_VEL_REPEAT=$v timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | head -3; done > gpurun_out/rep.levels.log 2>&1
for a in "cfg3 32 30" "cfg3 64 30" "cfg3 128 30" "cfg3 64 0" "cfg5 64 30"; do timeout 300 python tools/solve_probe.py $a; done > gpurun_out/rep.solve.log 2>&1
