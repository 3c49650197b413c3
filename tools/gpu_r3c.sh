#!/bin/bash
# round-2 final: full GPU suite, smoke, default bench, ncu of the pressure passes
mkdir -p gpurun_out
T=${1:-r3c}
python paper_1604_07994_b200/build.py > /dev/null
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/$T.pytest.log 2>&1; echo "exit $?" >> gpurun_out/$T.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T.smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/$T.bench.json 2> gpurun_out/$T.bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/$T.ref.json 2> gpurun_out/$T.ref.err
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled \
  -k regex:"k_stream<\(int\)0, \(int\)(3|4)>" -c 4 -o gpurun_out/$T.pp python tools/step_profiled.py cfg3 > gpurun_out/$T.ncu_pp.log 2>&1
