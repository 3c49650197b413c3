#!/bin/bash
# full state check: gpu tests, smoke, default bench (with cpu_baseline)
mkdir -p gpurun_out
T=${1:-r2t}
python paper_1604_07994_b200/build.py > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/$T.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T.smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
