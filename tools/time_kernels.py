"""Quick device timing of the hot kernels (CUDA events, L2 flushed between runs)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
import paper_1604_07994_b200 as stk

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 1
do_solve = not (len(sys.argv) > 4 and sys.argv[4] == "nosolve")
cfg = synth.get_config(name, n=n)
t0 = time.time()
cls, fcls = synth.element_classes(cfg)
print(f"classes {time.time()-t0:.1f}s", flush=True)
ctx = stk.StokesContext(n, "mod", cfg.faces)
ctx.set_kernel_mode(mode)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
lay = ctx.layout(0)
print("irregular", lay.n_irregular, lay.n_irregular / lay.n_vertices, flush=True)
x = torch.rand(lay.vec_len, dtype=torch.float64, device="cuda")
y = ctx.new_vector()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
V = (n + 1) ** 3


def timeit(fn, reps=10):
    ts = []
    for r in range(reps + 2):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return np.median(ts)


ms = timeit(lambda: ctx.apply(x, y))
print(f"apply: {ms:.3f} ms  {4*V/ms/1e6:.1f} GDoF/s  {65*V/ms/1e6:.0f} GB/s (65 B/vertex)", flush=True)
b = ctx.new_vector()
b.uniform_()
ms = timeit(lambda: ctx.residual(x, b, y))
print(f"residual: {ms:.3f} ms  {97*V/ms/1e6:.0f} GB/s (97 B/vertex)", flush=True)
ms = timeit(lambda: ctx.smooth(x, b, 1), reps=5)
print(f"uzawa step: {ms:.3f} ms  ({ms/6:.3f} per pass avg)", flush=True)
if not do_solve:
    sys.exit(0)
bb = ctx.load_nodal(synth.nodal_forcing(cfg)) if cfg.forcing == "nodal" else ctx.load_element(fcls, cfg.force_table)
torch.cuda.synchronize()
xs, rep = ctx.solve(bb, rtol=1e-8, max_cycles=60)
print(f"solve: cycles {rep.cycles} rho {rep.rho:.3f} rel {rep.rel_res:.2e} t {rep.t_total_s:.3f}s  "
      f"{rep.t_total_s/(4*V):.3e} s/DoF", flush=True)
print("hist", [f"{v:.2e}" for v in list(rep.res_hist)[:rep.cycles + 1]])
