#!/bin/bash
# One gpurun call: tests, smoke, short bench, launch list. Usage: tools/gpu_round.sh [tag]
tag=${1:-r}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/$tag.smi.txt 2>&1
nproc > gpurun_out/$tag.host.txt; lscpu | head -20 >> gpurun_out/$tag.host.txt; free -g >> gpurun_out/$tag.host.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$tag.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$tag.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag.smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/$tag.smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/$tag.bench.json 2> gpurun_out/$tag.bench.err; echo "bench exit $?" >> gpurun_out/$tag.bench.err
