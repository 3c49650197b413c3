for d in 0 1 2 3 4 7; do echo "== dbg $d"; STK_FUSED_DBG=$d timeout 100 python tools/trace_fused.py cfg2 128 32 2>&1 | grep "vel" | tail -3; done
