mkdir -p gpurun_out
tag=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse_level or uzawa or solve_matches" > gpurun_out/$tag.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$tag.pytest.log
timeout 200 python tools/prof_levels.py cfg2 128 > gpurun_out/$tag.levels.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$tag.bench.json 2> gpurun_out/$tag.bench.err
