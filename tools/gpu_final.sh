mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/fin.variants.log 2>&1; echo "exit $?" >> gpurun_out/fin.variants.log
timeout 200 python tools/prof_levels.py cfg2 128 > gpurun_out/fin.levels.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/fin.bench.json 2> gpurun_out/fin.bench.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin.ll.plain.json 2> gpurun_out/fin.ll.plain.err && \
timeout 1700 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin.launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin.ncu.log 2>&1
echo done
