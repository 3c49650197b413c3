#!/bin/bash
timeout 300 python tools/prof_levels.py cfg2 128 > gpurun_out/d10.levels.log 2>&1
timeout 300 python tools/prof_levels.py cfg4 512 >> gpurun_out/d10.levels.log 2>&1
