#!/bin/bash
# One gpurun call: tests, smoke, bench, per-level times, then ncu (launch list + one full capture).
# Usage: tools/gpu_full.sh tag [kernel-regex]
tag=${1:-r}; kre=${2:-k_stream}
bash tools/gpu_round.sh $tag
timeout 300 python tools/prof_levels.py cfg2 128 > gpurun_out/$tag.levels.log 2>&1
timeout 300 python tools/prof_apply.py cfg2 128 > gpurun_out/$tag.plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/$tag.launches.csv python tools/prof_apply.py cfg2 128 > gpurun_out/$tag.ncu1.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 3 \
   -o gpurun_out/$tag.prof python tools/prof_apply.py cfg2 128 > gpurun_out/$tag.ncu2.log 2>&1
echo done
