timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled or apply" > gpurun_out/regs.pytest.log 2>&1
for L in libstk.so libstk_r128.so libstk_r112.so; do echo "== $L"; STK_LIBNAME=$L timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | head -3; done > gpurun_out/regs.log 2>&1
