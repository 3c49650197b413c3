mkdir -p gpurun_out
for L in libstk.so libstk_minb3.so; do echo "== $L"; STK_LIBNAME=$L timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | head -9; done > gpurun_out/minb.log 2>&1
STK_LIBNAME=libstk_minb3.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled" > gpurun_out/minb.pytest.log 2>&1
