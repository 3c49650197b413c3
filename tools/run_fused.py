"""A few V-cycles at cfg2 (fused coarse levels) -- small driver for ncu."""
import sys
sys.path.insert(0, ".")
import torch
import synth
import paper_1604_07994_b200 as stk
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = synth.get_config(name, n=n)
cls, fcls = synth.element_classes(cfg)
ctx = stk.StokesContext(n, "mod", cfg.faces)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
b = ctx.load_nodal(synth.nodal_forcing(cfg))
x = ctx.new_vector()
for _ in range(2):
    ctx.vcycle(b, x)
torch.cuda.synchronize()
print("ok")
