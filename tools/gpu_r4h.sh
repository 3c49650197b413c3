#!/bin/bash
# bench with the clock sampler started before the warm-up (both arms)
mkdir -p gpurun_out
T=${1:-r4h}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$T.bench_ref.json 2> gpurun_out/$T.bench_ref.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/$T.bench2.json 2> gpurun_out/$T.bench2.err
