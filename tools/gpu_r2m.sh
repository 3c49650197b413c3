#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2m}
python paper_1604_07994_b200/build.py -v 2> gpurun_out/$T.ptxas.log > /dev/null
timeout 300 python -m pytest tests/test_gpu_loopback.py -q > gpurun_out/$T.loop.log 2>&1; echo "exit $?" >> gpurun_out/$T.loop.log
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "solve" > gpurun_out/$T.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T.pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 600 python tools/form_compare.py 128 > gpurun_out/$T.forms.json 2> gpurun_out/$T.forms.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_stream" -c 4 \
   -o gpurun_out/$T.full python tools/prof_apply.py cfg3 256 > gpurun_out/$T.ncu.log 2>&1
