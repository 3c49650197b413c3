"""Operator-apply table over the BASELINE workloads on one B200: per config
the apply time (CUDA events, L2 flushed before every launch), GDoF/s (DoF = 4 (n+1)^3, R21),
HBM GB/s by the 65 B/vertex of SURVEY 8(d) and the fraction of the measured peak.
cfg5 (n = 1024 on 8 GPUs) runs here at n = 512, the size of one GPU's share.
usage: apply_table.py > profiles/r02_apply_table.json"""
import json
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import synth
import paper_1604_07994_b200 as stk

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for name, n in (("cfg1", 16), ("cfg2", 128), ("cfg3", 256), ("cfg4", 512), ("cfg5", 512), ("cols", 512)):
    cfg = synth.get_config(name, n=n)
    cls, _ = synth.element_classes(cfg)
    ctx = stk.StokesContext(n, "mod", cfg.faces)
    ctx.set_viscosity(cls, cfg.class_mu)
    ctx.assemble()
    lay = ctx.layout(0)
    x = torch.rand(lay.vec_len, dtype=torch.float64, device="cuda")
    y = ctx.new_vector()
    for _ in range(3):
        ctx.apply(x, y)
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.apply(x, y)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = float(np.median(ms))
    V = (n + 1) ** 3
    row = {"workload": name, "n": n, "dofs": 4 * V, "apply_ms": round(t, 4), "gdof_s": round(4 * V / t / 1e6, 2),
           "hbm_gbs": round(65 * V / t / 1e6, 1), "frac_of_peak": round(65 * V / t / 1e6 / peak, 4),
           "tiled_kernels": n >= 64}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del ctx, x, y
    torch.cuda.empty_cache()
