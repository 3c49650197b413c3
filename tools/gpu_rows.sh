mkdir -p gpurun_out
tag=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse_level or uzawa or solve_matches" > gpurun_out/$tag.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$tag.pytest.log
for lpr in 1 4 16 0; do echo "== STK_ROW_LPR=$lpr"; STK_ROW_LPR=$lpr timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | tail -8; done > gpurun_out/$tag.levels.log 2>&1
