#!/bin/bash
# final-candidate state check: full GPU suite, smoke, bench (both arms)
mkdir -p gpurun_out
T=${1:-r4f}
python paper_1604_07994_b200/build.py > /dev/null
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/$T.gputest.log 2>&1; echo "exit $?" >> gpurun_out/$T.gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T.smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$T.bench_ref.json 2> gpurun_out/$T.bench_ref.err
