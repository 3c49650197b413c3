"""Per-(op, level) device time of V-cycles (stk profile API, CUDA events)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import synth
import paper_1604_07994_b200 as stk

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = synth.get_config(name, n=n)
cls, fcls = synth.element_classes(cfg)
kry = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ctx = stk.StokesContext(n, "mod", cfg.faces)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
b = ctx.load_nodal(synth.nodal_forcing(cfg)) if cfg.forcing == "nodal" else ctx.load_element(fcls, cfg.force_table)
x = ctx.new_vector()
for _ in range(2):
    ctx.vcycle(b, x)
torch.cuda.synchronize()
ctx.profile(2)
ctx.profile_reset()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
ncyc = 3
for _ in range(ncyc):
    ctx.vcycle(b, x)
e1.record()
torch.cuda.synchronize()
print(f"{name} n={n}: {e0.elapsed_time(e1)/ncyc:.3f} ms per V-cycle (with profiling events)")
nlev = int(np.log2(n // 4)) + 1
tot = 0
for lv in range(nlev):
    row = []
    for op in ctx.PROFILE_OPS:
        cnt, ms = ctx.profile_read(op, lv)
        if cnt:
            row.append(f"{op}:{cnt//ncyc}x{ms/cnt*1e3:.1f}us")
            tot += ms
    print(f"  level {lv} (n={n >> lv}): " + "  ".join(row))
print(f"  sum of op times {tot/ncyc:.3f} ms per cycle")
ctx.profile(False)
torch.cuda.synchronize()
e0.record()
for _ in range(ncyc):
    ctx.vcycle(b, x)
e1.record()
torch.cuda.synchronize()
print(f"  without profiling: {e0.elapsed_time(e1)/ncyc:.3f} ms per V-cycle")
for rn, fz in ((0, 0), (16, 0), (32, 0), (64, 0), (16, 8), (16, 16), (32, 32)):
    ctx.set_row_n(rn)
    ctx.set_fuse_n(fz)
    for _ in range(2):
        ctx.vcycle(b, x)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(ncyc):
        ctx.vcycle(b, x)
    e1.record()
    torch.cuda.synchronize()
    print(f"  row_n={rn} fuse_n={fz} (row level {ctx.row_level()}, fused level {ctx.fused_level()}): "
          f"{e0.elapsed_time(e1)/ncyc:.3f} ms per V-cycle")
