"""Solver-parameter sweep on one config: iterations and device time of the solve for
V_var smoothing increments, GMRES restart lengths and row-kernel thresholds.
usage: solve_sweep.py cfg n"""
import sys
import itertools
sys.path.insert(0, ".")
import torch
import synth
import paper_1604_07994_b200 as stk
name, n = sys.argv[1], int(sys.argv[2])
cfg = synth.get_config(name, n=n)
cls, fcls = synth.element_classes(cfg)
f = synth.nodal_forcing(cfg) if cfg.forcing == "nodal" else None
for nu, nu_inc, kry in [(3, 2, 30), (3, 1, 30), (3, 0, 30), (2, 1, 30), (3, 2, 20), (4, 0, 30), (2, 2, 30)]:
    ctx = stk.StokesContext(n, "mod", cfg.faces, nu_pre=nu, nu_post=nu, nu_inc=nu_inc, krylov=kry)
    ctx.set_viscosity(cls, cfg.class_mu)
    ctx.assemble()
    b = ctx.load_nodal(f) if f is not None else ctx.load_element(fcls, cfg.force_table)
    x = ctx.new_vector()
    ctx.solve(b, x, rtol=1e-8, max_cycles=300)
    ts = []
    for _ in range(2):
        x.zero_()
        x, rep = ctx.solve(b, x, rtol=1e-8, max_cycles=300)
        ts.append(rep.t_total_s)
    print(f"{name} n={n} nu={nu} nu_inc={nu_inc} krylov={kry}: its={rep.cycles} rel={rep.rel_res:.2e} "
          f"solve={min(ts)*1e3:.1f} ms ({min(ts)/max(rep.cycles,1)*1e3:.2f} ms/it)", flush=True)
    ctx.close()
    torch.cuda.empty_cache()
