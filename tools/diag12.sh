#!/bin/bash
timeout 300 python tools/prof_levels.py cfg2 128 > gpurun_out/d12.levels.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/d12.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/d12.pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/d12.bench.json 2> gpurun_out/d12.bench.err
