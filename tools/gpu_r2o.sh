#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2o}
python paper_1604_07994_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "uzawa or tiled or solve_on_tiled" > gpurun_out/$T.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T.pytest.log
timeout 300 python -m pytest tests/test_gpu_variants.py tests/test_gpu_loopback.py -q > gpurun_out/$T.var.log 2>&1; echo "exit $?" >> gpurun_out/$T.var.log
timeout 300 python tools/prof_levels.py cfg3 256 > gpurun_out/$T.levels.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
