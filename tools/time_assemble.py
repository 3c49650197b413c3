"""Time stk_assemble (and set_viscosity + assemble) on cfg2 with CUDA events."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import synth
import paper_1604_07994_b200 as stk
cfg = synth.get_config("cfg2")
cls, fcls = synth.element_classes(cfg)
ctx = stk.StokesContext(cfg.n, "mod", cfg.faces)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
b = ctx.load_nodal(synth.nodal_forcing(cfg))
x = ctx.new_vector()
ctx.solve(b, x, rtol=1e-8)
for mode in ("assemble", "set+assemble", "set+assemble+solve"):
    ts = []
    for r in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode != "assemble":
            ctx.set_viscosity(cls, cfg.class_mu)
        ctx.assemble()
        if mode.endswith("solve"):
            x.zero_()
            ctx.solve(b, x, rtol=1e-8)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{mode:22s} ms: " + " ".join(f"{t:.2f}" for t in ts))
