"""Minimal driver for ncu: a few applies + one Uzawa step.  usage: prof_apply.py [cfg] [n]"""
import sys
sys.path.insert(0, ".")
import torch
import synth
import paper_1604_07994_b200 as stk
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = synth.get_config(name, n=n)
cls, _ = synth.element_classes(cfg)
ctx = stk.StokesContext(n, "mod", cfg.faces)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
lay = ctx.layout(0)
x = torch.rand(lay.vec_len, dtype=torch.float64, device="cuda")
b = torch.rand(lay.vec_len, dtype=torch.float64, device="cuda")
y = ctx.new_vector()
for _ in range(3):
    ctx.apply(x, y)
ctx.smooth(x, b, 1)
torch.cuda.synchronize()
print("ok")
