mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled or apply or uzawa" > gpurun_out/slack.pytest.log 2>&1
for L in libstk.so libstk_slack0.so libstk_slack2.so; do echo "== $L"; STK_LIBNAME=$L timeout 200 python tools/prof_levels.py cfg2 128 2>&1 | head -9; done > gpurun_out/pref.log 2>&1
