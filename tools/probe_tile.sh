#!/bin/bash
timeout 30 ./tools/probe_tma_neg > gpurun_out/probe_tile3.log 2>&1
for a in "32 8 1 1 0 0" "32 8 1 1 1 1" "32 8 1 1 0 1" "34 10 1 1 0 0" "34 10 1 1 0 1"; do
  timeout 30 ./tools/probe_tma_tile $a >> gpurun_out/probe_tile3.log 2>&1
done
