"""Convergence probe: solve a config at size n with the V-cycle (krylov=0) or GMRES(m)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import synth
import paper_1604_07994_b200 as stk
name, n, kry = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cmu = sys.argv[4] if len(sys.argv) > 4 else "arith"
nc = int(sys.argv[5]) if len(sys.argv) > 5 else 4
cfg = synth.get_config(name, n=n)
cls, fcls = synth.element_classes(cfg)
ctx = stk.StokesContext(n, "mod", cfg.faces, krylov=kry, coarse_mu=cmu, n_coarse=nc)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
b = ctx.load_nodal(synth.nodal_forcing(cfg)) if cfg.forcing == "nodal" else ctx.load_element(fcls, cfg.force_table)
x, rep = ctx.solve(b, rtol=1e-8, max_cycles=200)
h = [rep.res_hist[i] for i in range(min(rep.cycles, 256))]
print(f"{name} n={n} krylov={kry} coarse_mu={cmu} n_coarse={nc}: its={rep.cycles} rel={rep.rel_res:.3e} t={rep.t_total_s:.3f}s hist[0:8]={np.array(h[:8])} last={h[-3:]}")
r, nr = ctx.residual(x, b, norms=True)
nb = ctx.norms(b)
print(f"  residual per field (u1,u2,u3,p): {np.sqrt(nr[:4])}  |b| per field: {np.sqrt(nb[:4])}")
