#!/bin/bash
# coarse MINRES parity + GMRES(Z) solve tests; cfg3 bench restart sweep; rho fix; coarse compare
mkdir -p gpurun_out
T=${1:-r2w}
python paper_1604_07994_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_coarse_minres.py tests/test_gpu_loopback.py -q -x > gpurun_out/$T.mr.log 2>&1; echo "exit $?" >> gpurun_out/$T.mr.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "solve" > gpurun_out/$T.solve.log 2>&1; echo "exit $?" >> gpurun_out/$T.solve.log
for m in 30 20 12 8; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --krylov $m > gpurun_out/$T.bench_k$m.json 2> gpurun_out/$T.bench_k$m.err
done
timeout 900 python tools/coarse_compare.py cols 256 > gpurun_out/$T.coarse_cols.json 2> gpurun_out/$T.coarse_cols.err
timeout 900 python tools/cols_study.py 8 512 40 128 > gpurun_out/$T.study.json 2> gpurun_out/$T.study.err
