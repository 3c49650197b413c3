set -x
timeout 600 python -m pytest tests -m gpu -q -k "solve or tiled" > gpurun_out/d1.pytest.log 2>&1
for e in "" "STK_SKIP_IRR=1" "STK_NO_TMA=1"; do
  env $e timeout 300 python tools/time_kernels.py cfg2 128 1 nosolve >> gpurun_out/d1.time.log 2>&1
done
timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d1.time.log 2>&1
STK_SKIP_IRR=1 timeout 300 python tools/time_kernels.py cfg4 512 1 nosolve >> gpurun_out/d1.time.log 2>&1
timeout 300 python tools/prof_apply.py cfg2 128 > gpurun_out/d1.plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream -c 4 -o gpurun_out/d1_apply python tools/prof_apply.py cfg2 128 > gpurun_out/d1.ncu.log 2>&1
