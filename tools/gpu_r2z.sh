#!/bin/bash
# cfg4 stagnation probes; list-row stencil skipping check (cols parity + bench)
mkdir -p gpurun_out
T=${1:-r2z}
python paper_1604_07994_b200/build.py > /dev/null
for v in "256 0" "256 100" "128 30" "192 30"; do
  timeout 400 python tools/solve_probe.py cfg4 $v >> gpurun_out/$T.cfg4probe.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -k "cols or listx or apply" > gpurun_out/$T.cols.log 2>&1; echo "exit $?" >> gpurun_out/$T.cols.log
timeout 900 python bench.py --workload cols --n 256 --steps 3 --no-cpu-baseline > gpurun_out/$T.cols256.json 2> gpurun_out/$T.cols256.err
