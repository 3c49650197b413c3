mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q -k "tiled or uzawa or apply or switch or solve_matches" > gpurun_out/chk.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/chk.pytest.log
timeout 200 python tools/time_assemble.py > gpurun_out/chk.asm.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/chk.bench.json 2> gpurun_out/chk.bench.err
