#!/bin/bash
# full GPU test suite (durations), smoke, bench at cfg3 n=256
mkdir -p gpurun_out
T=${1:-r2j}
python paper_1604_07994_b200/build.py > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/$T.smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/$T.smoke.log
timeout 300 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/$T.loop.log 2>&1; echo "exit $?" >> gpurun_out/$T.loop.log
timeout 1200 python -m pytest tests -m gpu -q --durations=30 --deselect tests/test_gpu_loopback.py > gpurun_out/$T.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T.pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
