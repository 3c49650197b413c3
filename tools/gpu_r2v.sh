#!/bin/bash
# free-slip parity (incl. loopback), full GPU suite, NEXT-1 study (cols)
mkdir -p gpurun_out
T=${1:-r2v}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -q -k cols > gpurun_out/$T.cols.log 2>&1; echo "exit $?" >> gpurun_out/$T.cols.log
timeout 1500 python tools/cols_study.py 256 512 60 > gpurun_out/$T.study.json 2> gpurun_out/$T.study.err
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/$T.pytest.log 2>&1; echo "exit $?" >> gpurun_out/$T.pytest.log
