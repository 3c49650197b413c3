mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "uzawa or solve or coarse_level or tiled_smoother" > gpurun_out/gj.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gj.pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gj.bench.json 2> gpurun_out/gj.bench.err
