"""NEXT-2: the paper's coarse-grid strategy against the direct coarse
solve on one B200: per V-cycle time, asymptotic rate rho (zero rhs, random start,
rescaled and gauged every cycle), and V-cycles to 1e-8, for coarse grids
n_c = 4, 8 and the paper's L = 2 grid n_c = 16 (19,652 DoF).

    python tools/coarse_compare.py [workload=cols] [n=256] [its=20] [cg_its=4]
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import synth
import paper_1604_07994_b200 as stk

name = sys.argv[1] if len(sys.argv) > 1 else "cols"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
its = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cg = int(sys.argv[4]) if len(sys.argv) > 4 else 4
cfg = synth.get_config(name, n=n)
cls, fcls = synth.element_classes(cfg)
out = {"workload": name, "n": n, "dofs": cfg.dofs, "minres_its": its, "cg_its": cg, "runs": []}
for nc, kind in ((4, "direct"), (8, "direct"), (4, "minres"), (8, "minres"), (16, "minres")):
    ctx = stk.StokesContext(n, "mod", cfg.faces, n_coarse=nc)
    ctx.set_viscosity(cls, cfg.class_mu)
    ctx.assemble()
    if kind == "minres":
        ctx.set_coarse_solver("minres", its, cg)
    b = ctx.load_nodal(synth.nodal_forcing(cfg)) if cfg.forcing == "nodal" else ctx.load_element(fcls, cfg.force_table)
    xv = ctx.new_vector()
    for _ in range(2):
        ctx.vcycle(b, xv)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        ctx.vcycle(b, xv)
    e1.record()
    torch.cuda.synchronize()
    t_cycle = e0.elapsed_time(e1) / 10
    x, rep = ctx.solve(b, rtol=1e-8, max_cycles=100)
    z = ctx.new_vector()
    lay = ctx.layout(0)
    rng = np.random.default_rng(1)
    xr = ctx.import_(rng.uniform(-1, 1, (4, lay.n_vertices)))
    prev = np.sqrt(ctx.residual(xr, z, norms=True)[1][4])
    rates = []
    for _ in range(40):
        xr.mul_(1.0 / prev)
        ctx.vcycle(z, xr)
        ctx.gauge(xr)
        cur = np.sqrt(ctx.residual(xr, z, norms=True)[1][4])
        rates.append(cur)
        prev = cur
    ctx.profile(2)
    ctx.profile_reset()
    ctx.vcycle(b, xv)
    c_cnt, c_ms = ctx.profile_read("coarse", -1)
    ctx.profile(0)
    row = {"n_coarse": nc, "coarse": kind, "ms_per_cycle": round(t_cycle, 3), "coarse_solve_ms": round(c_ms, 4),
           "cycles_to_1e-8": rep.cycles, "rel_res": rep.rel_res, "rho_geo_last10": round(float(np.prod(rates[-10:]) ** 0.1), 4)}
    out["runs"].append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
    ctx.close()
print(json.dumps(out, indent=1))
