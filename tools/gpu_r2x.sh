#!/bin/bash
# full GPU suite + smoke + default bench (cfg3) + cfg5/cfg4/cols bench lines
mkdir -p gpurun_out
T=${1:-r2x}
python paper_1604_07994_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$T.pytest.log 2>&1; echo "exit $?" >> gpurun_out/$T.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T.smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 900 python bench.py --workload cfg5 --n 256 --krylov 12 --steps 3 --no-cpu-baseline > gpurun_out/$T.cfg5_k12.json 2> gpurun_out/$T.cfg5_k12.err
timeout 900 python bench.py --workload cfg5 --n 256 --krylov 30 --steps 3 --no-cpu-baseline > gpurun_out/$T.cfg5_k30.json 2> gpurun_out/$T.cfg5_k30.err
timeout 900 python bench.py --workload cols --n 512 --steps 3 --no-cpu-baseline > gpurun_out/$T.cols512.json 2> gpurun_out/$T.cols512.err
timeout 1200 python bench.py --workload cfg4 --n 512 --krylov 12 --steps 2 --no-cpu-baseline > gpurun_out/$T.cfg4_512.json 2> gpurun_out/$T.cfg4_512.err
