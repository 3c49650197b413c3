#!/bin/bash
# free-slip parity, full GPU suite, cfg3 bench (CGS1 GMRES), cols bench, level profile
mkdir -p gpurun_out
T=${1:-r2u}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -q -k cols > gpurun_out/$T.cols.log 2>&1; echo "exit $?" >> gpurun_out/$T.cols.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 600 python bench.py --workload cols --n 256 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T.cols256.json 2> gpurun_out/$T.cols256.err
timeout 300 python tools/prof_levels.py cfg3 256 > gpurun_out/$T.levels.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/$T.pytest.log 2>&1; echo "exit $?" >> gpurun_out/$T.pytest.log
