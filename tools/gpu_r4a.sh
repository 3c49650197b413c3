#!/bin/bash
# session-6 state check: fp64 probes, full GPU suite, smoke, bench (both arms)
mkdir -p gpurun_out
T=${1:-r4a}
python paper_1604_07994_b200/build.py > /dev/null
nvcc -arch=sm_100a -O3 -o /tmp/probe_fp64 tools/probe_fp64.cu && /tmp/probe_fp64 > gpurun_out/$T.probe_fp64.log 2>&1
nvcc -arch=sm_100a -O3 -o /tmp/probe_dfma tools/probe_dfma.cu && /tmp/probe_dfma > gpurun_out/$T.probe_dfma.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/$T.gputest.log 2>&1; echo "exit $?" >> gpurun_out/$T.gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T.smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$T.bench_ref.json 2> gpurun_out/$T.bench_ref.err
