#!/bin/bash
# cluster MINRES parity + coarse compare; bench (profiling out of the timed steps); cfg4 probes;
# ncu launch list of one bench step; ncu full of the level-0 kernels
mkdir -p gpurun_out
T=${1:-r2y}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_coarse_minres.py -q > gpurun_out/$T.mr.log 2>&1; echo "exit $?" >> gpurun_out/$T.mr.log
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
for v in "arith 4" "harmonic 4" "arith 8" "harmonic 8"; do
  timeout 300 python tools/solve_probe.py cfg4 256 30 $v >> gpurun_out/$T.cfg4probe.log 2>&1
done
timeout 900 python tools/coarse_compare.py cols 256 > gpurun_out/$T.coarse_cols.json 2> gpurun_out/$T.coarse_cols.err
timeout 600 python tools/step_profiled.py cfg3 > gpurun_out/$T.step.log 2>&1
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/$T.launches.csv python tools/step_profiled.py cfg3 > gpurun_out/$T.ncu_ll.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"k_stream|k_listx|k_gs_pass|k_prolong|k_restrict" -c 12 -o gpurun_out/$T.full python tools/step_profiled.py cfg3 > gpurun_out/$T.ncu_full.log 2>&1
gzip -f gpurun_out/$T.launches.csv
