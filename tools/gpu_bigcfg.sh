mkdir -p gpurun_out
timeout 900 python bench.py --workload cfg3 --krylov 30 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/big.cfg3.json 2> gpurun_out/big.cfg3.err
timeout 1200 python bench.py --workload cfg4 --krylov 30 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/big.cfg4.json 2> gpurun_out/big.cfg4.err
timeout 300 python tools/prof_levels.py cfg4 512 > gpurun_out/big.levels4.log 2>&1
