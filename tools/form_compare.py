"""a4: the three viscous forms on BASELINE configs[1] (cfg2: plane interface with
mu1/mu2 = 1e3, traction-free top), as in the paper's Table timeANDconv:
per-cycle time and asymptotic rate rho of the V_var(3,3) Uzawa multigrid, iterations
to 1e-8, and the solution differences mod - sym and grad - sym.

    python tools/form_compare.py [n=128] > profiles/r02_form_compare.json

rho is measured the paper's way: b = 0, random x0, the residual rescaled to
1 after every cycle, rho = the reduction of the last of `rho_cycles` cycles.
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import synth
import paper_1604_07994_b200 as stk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rho_cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = synth.get_config("cfg2", n=n)
cls, _ = synth.element_classes(cfg)
f = synth.nodal_forcing(cfg)
out = {"config": f"cfg2 n={n} (BASELINE configs[1]), {cfg.dofs} DoF", "forms": {}}
sols = {}
for form in ("mod", "sym", "grad"):
    nc = 4 if form == "sym" else 2
    ctx = stk.StokesContext(n, form, cfg.faces, ncolors_u=nc)
    ctx.set_viscosity(cls, cfg.class_mu)
    ctx.assemble()
    b = ctx.load_nodal(f)
    x = ctx.new_vector()
    ctx.solve(b, x, rtol=1e-8, max_cycles=100)          # warm-up (graph capture)
    x.zero_()
    x, rep = ctx.solve(b, x, rtol=1e-8, max_cycles=100)
    sols[form] = ctx.export(x)
    # per-cycle time: 10 cycles, CUDA events
    xv = ctx.new_vector()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        ctx.vcycle(b, xv)
    e1.record()
    torch.cuda.synchronize()
    t_cycle = e0.elapsed_time(e1) / 10
    # asymptotic rate: zero rhs, random start, rescaled every cycle
    z = ctx.new_vector()
    lay = ctx.layout(0)
    rng = np.random.default_rng(1)
    xr = ctx.import_(rng.uniform(-1, 1, (4, lay.n_vertices)))
    prev = np.sqrt(ctx.residual(xr, z, norms=True)[1][4])
    rates = []
    for _ in range(rho_cycles):
        xr.mul_(1.0 / prev)
        ctx.vcycle(z, xr)
        ctx.gauge(xr)      # the constant pressure is never reduced: project it out
        cur = np.sqrt(ctx.residual(xr, z, norms=True)[1][4])
        rates.append(cur)          # residual of a unit-residual start
        prev = cur
    out["forms"][form] = {"iterations_to_1e-8": rep.cycles, "rel_res": rep.rel_res,
                          "solve_ms": rep.t_total_s * 1e3, "ms_per_cycle": round(t_cycle, 3),
                          "rho_last": round(float(rates[-1]), 4),
                          "rho_geo_last10": round(float(np.prod(rates[-10:]) ** 0.1), 4),
                          "ncolors_u": nc, "n_irregular_rows": int(lay.n_irregular)}
    ctx.close()
ref = sols["sym"]
for form in ("mod", "grad"):
    d = sols[form] - ref
    out["forms"][form]["diff_vs_sym"] = {
        "velocity_rel_l2": float(np.linalg.norm(d[:3]) / np.linalg.norm(ref[:3])),
        "pressure_rel_l2": float(np.linalg.norm(d[3]) / np.linalg.norm(ref[3])),
        "velocity_max_abs": float(np.abs(d[:3]).max()), "velocity_max": float(np.abs(ref[:3]).max())}
out["speedup_mod_over_sym_per_cycle"] = round(out["forms"]["sym"]["ms_per_cycle"] / out["forms"]["mod"]["ms_per_cycle"], 3)
out["paper"] = {"table": "timeANDconv (P:1312-1330), Intel 2x Xeon E5-2699, columns problem with free slip",
                "L5_n128_T_cycle_s": {"strain": 1.18, "mod": 1.12, "grad": 1.34},
                "L5_rho": {"strain": 0.296, "mod": 0.244, "grad": 0.240}}
print(json.dumps(out, indent=1))
