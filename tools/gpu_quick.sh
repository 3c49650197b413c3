mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse_level or uzawa or tiled_smoother or solve_matches" > gpurun_out/${1:-q}.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${1:-q}.pytest.log
timeout 300 python tools/prof_levels.py cfg2 128 > gpurun_out/${1:-q}.levels.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${1:-q}.bench.json 2> gpurun_out/${1:-q}.bench.err
