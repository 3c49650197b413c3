mkdir -p gpurun_out
tag=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled or apply or uzawa" > gpurun_out/$tag.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$tag.pytest.log
for v in 1 0; do echo "== STK_LIST_EXPLICIT=$v"; STK_LIST_EXPLICIT=$v timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | head -9; done > gpurun_out/$tag.levels.log 2>&1
