#!/bin/bash
timeout 300 python tools/prof_apply.py cfg2 128 > gpurun_out/d14.plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream" -s 3 -c 2 -o gpurun_out/d14_vel128 python tools/prof_apply.py cfg2 128 > gpurun_out/d14.ncu.log 2>&1
