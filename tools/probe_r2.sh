timeout 60 ./tools/probe_tma_sweep 36 12 > gpurun_out/probe_sw.log 2>&1
timeout 60 ./tools/probe_tma_sweep 34 10 >> gpurun_out/probe_sw.log 2>&1
timeout 60 ./tools/probe_tma_sweep 36 10 >> gpurun_out/probe_sw.log 2>&1
