#!/bin/bash
timeout 300 python tools/prof_levels.py cfg2 128 > gpurun_out/d13.levels.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/d13.bench.json 2> gpurun_out/d13.bench.err
timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve > gpurun_out/d13.time.log 2>&1
