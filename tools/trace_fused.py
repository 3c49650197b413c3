"""Per-phase trace of the fused coarse V-cycle (STK_FUSED_TRACE=1)."""
import os, sys
os.environ["STK_FUSED_TRACE"] = "1"
os.environ["STK_NO_GRAPH"] = "1"
sys.path.insert(0, ".")
import torch
import synth
import paper_1604_07994_b200 as stk
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
fz = int(sys.argv[3]) if len(sys.argv) > 3 else 32
cfg = synth.get_config(name, n=n)
cls, fcls = synth.element_classes(cfg)
ctx = stk.StokesContext(n, "mod", cfg.faces)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
ctx.set_fuse_n(fz)
b = ctx.load_nodal(synth.nodal_forcing(cfg))
x = ctx.new_vector()
for _ in range(3):
    ctx.vcycle(b, x)
    torch.cuda.synchronize()
