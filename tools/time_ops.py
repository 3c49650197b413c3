"""Level-0 kernel times at a config (CUDA events, profile mode 2): apply, residual, a
velocity colour pass, pressure passes 1 and 2 -- for kernel-variant experiments.
usage: time_ops.py [cfg3] [256] [label]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import synth
import paper_1604_07994_b200 as stk
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
label = sys.argv[3] if len(sys.argv) > 3 else ""
cfg = synth.get_config(name, n=n)
cls, fcls = synth.element_classes(cfg)
ctx = stk.StokesContext(n, "mod", cfg.faces)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
b = ctx.load_nodal(synth.nodal_forcing(cfg)) if cfg.forcing == "nodal" else ctx.load_element(fcls, cfg.force_table)
x = ctx.new_vector()
y = ctx.new_vector()
for _ in range(2):
    ctx.vcycle(b, x)
    ctx.apply(x, y)
torch.cuda.synchronize()
ctx.profile(2)
ctx.profile_reset()
for _ in range(3):
    ctx.vcycle(b, x)
    for _ in range(5):
        ctx.apply(x, y)
torch.cuda.synchronize()
out = []
for op in ("apply", "residual", "vel_pass", "p_pass1", "p_pass2"):
    c, ms = ctx.profile_read(op, 0)
    out.append(f"{op} {1e3 * ms / max(c, 1):.1f}us")
ctx.profile(0)
print(f"{label} {name} n={n} level 0: " + "  ".join(out))
