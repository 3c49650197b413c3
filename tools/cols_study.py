"""NEXT-1: the paper's own workload -- viscosity columns with free slip on all faces
(mu2 = 10 in two corner columns, f = (0,0,-cos 2pi x cos 2pi y sin pi z)),
on one B200, next to the paper's tables:

* consistency (lumped-mass L2 norms; Tables columns-laplace-p1p1 / columns-stencil-p1p1): the
  relative differences of the gradient-based and the modified-stencil solutions to the
  strain-based one in L2 (velocity), the V-norm (here the mu = 1 gradient energy
  seminorm) and L2 (pressure), levels L = 2..6 (n = 4 * 2^L = 16..256);
* multigrid (Table timeANDconv): time of one V_var(3,3) cycle and the
  asymptotic rate rho (zero rhs, random start, residual rescaled every cycle) at
  L = 5, 6, 7 (n = 128, 256, 512) for the three forms.

    python tools/cols_study.py [max_consistency_n=256] [max_mg_n=512] [rho_cycles=60]
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import synth
import paper_1604_07994_b200 as stk

nmax_c = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nmin_m = int(sys.argv[4]) if len(sys.argv) > 4 else 128
nmax_m = int(sys.argv[2]) if len(sys.argv) > 2 else 512
rho_cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 60
FORMS = ("sym", "mod", "grad")
PAPER = {
    "grad_vs_sym": {"L2": [7.4550e-02, 3.0104e-02, 2.1227e-02, 2.0227e-02, 2.0098e-02],
                    "V": [9.2581e-02, 6.0398e-02, 4.7364e-02, 4.3246e-02, 4.2121e-02],
                    "p": [2.7609e01, 1.8003e-01, 1.1179e-01, 8.0546e-02, 6.9997e-02]},
    "mod_vs_sym": {"L2": [1.3890e-02, 4.2414e-03, 1.1370e-03, 2.9449e-04, 7.5985e-05],
                   "V": [2.4189e-02, 1.2312e-02, 6.2303e-03, 3.1918e-03, 1.6675e-03],
                   "p": [7.7949e-02, 4.8195e-02, 2.5287e-02, 1.3274e-02, 6.8175e-03]},
    "levels": [2, 3, 4, 5, 6],
    "timeANDconv": {"hardware": "2x Xeon E5-2699 (32 cores), HHG, coarse grid L=2 (19,652 DoF) MINRES",
                    "T_cycle_s": {"5": {"sym": 1.18, "mod": 1.12, "grad": 1.34},
                                  "6": {"sym": 3.02, "mod": 2.45, "grad": 2.64},
                                  "7": {"sym": 13.95, "mod": 9.04, "grad": 9.26},
                                  "8": {"sym": 93.74, "mod": 54.08, "grad": 54.22}},
                    "rho": {"5": {"sym": 0.296, "mod": 0.244, "grad": 0.240},
                            "6": {"sym": 0.280, "mod": 0.242, "grad": 0.240},
                            "7": {"sym": 0.263, "mod": 0.241, "grad": 0.241},
                            "8": {"sym": 0.255, "mod": 0.241, "grad": 0.241}}},
}


def ctx_for(n, form, cfg, cls):
    ctx = stk.StokesContext(n, form, cfg.faces, ncolors_u=4 if form == "sym" else 2)
    ctx.set_viscosity(cls, cfg.class_mu)
    ctx.assemble()
    return ctx


def lumped_w(n):
    """trapezoidal (lumped-mass) vertex weights h^3 * prod over axes (1/2 on a face)."""
    w1 = np.ones(n + 1)
    w1[0] = w1[-1] = 0.5
    return (np.einsum("k,j,i->kji", w1, w1, w1) / n ** 3).reshape(-1)


out = {"workload": "cols: viscosity columns, free slip on all faces (P:772-774, P:719)", "consistency": [],
       "multigrid": [], "paper": PAPER}

# ---- consistency table --------------------------------------------------------------
n = 16
while n <= nmax_c:
    cfg = synth.get_config("cols", n=n)
    cls, _ = synth.element_classes(cfg)
    f = synth.nodal_forcing(cfg)
    sol, its = {}, {}
    for form in FORMS:
        ctx = ctx_for(n, form, cfg, cls)
        b = ctx.load_nodal(f)
        x, rep = ctx.solve(b, rtol=1e-11, max_cycles=200)
        sol[form] = ctx.export(x)
        its[form] = (rep.cycles, rep.rel_res)
        ctx.close()
    # norms: discrete L2 by the lumped mass (trapezoidal weights); V-norm = the mu = 1
    # gradient energy seminorm (library apply, block A, free-slip context)
    wl = lumped_w(n)
    ones = np.zeros(6 * n ** 3, dtype=np.uint8)
    cv = stk.StokesContext(n, "grad", cfg.faces)
    cv.set_viscosity(ones, (1.0,))
    cv.assemble()

    def l2(d):
        return float(np.sum(wl * d[:3] ** 2))

    def pl2(p):
        return float(np.sum(wl * p ** 2))

    def vnorm2(d):
        dv = np.zeros_like(d)
        dv[:3] = d[:3]
        return float(np.sum(cv.export(cv.apply(cv.import_(dv), blocks=1))[:3] * d[:3]))

    row = {"n": n, "level": int(round(np.log2(n // 4))), "iterations": its}
    ref = sol["sym"]
    for form in ("mod", "grad"):
        d = sol[form] - ref
        row[f"{form}_vs_sym"] = {
            "L2": (l2(d) / l2(ref)) ** 0.5,
            "V": (vnorm2(d) / vnorm2(ref)) ** 0.5,
            "p": (pl2(d[3]) / pl2(ref[3])) ** 0.5}
    cv.close()
    out["consistency"].append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
    n *= 2
for key in ("mod_vs_sym", "grad_vs_sym"):
    for q in ("L2", "V", "p"):
        v = [r[key][q] for r in out["consistency"]]
        out.setdefault("rates", {}).setdefault(key, {})[q] = [round(float(np.log2(a / b)), 3)
                                                                for a, b in zip(v[:-1], v[1:])]

# ---- time per V-cycle and asymptotic rate ---------------------------------------------
n = nmin_m
while n <= nmax_m:
    cfg = synth.get_config("cols", n=n)
    cls, _ = synth.element_classes(cfg)
    row = {"n": n, "level": int(round(np.log2(n // 4))), "dofs": cfg.dofs}
    for form in FORMS:
        ctx = ctx_for(n, form, cfg, cls)
        b = ctx.load_nodal(synth.nodal_forcing(cfg))
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
        z = ctx.new_vector()
        lay = ctx.layout(0)
        rng = np.random.default_rng(1)
        xr = ctx.import_(rng.uniform(-1, 1, (4, lay.n_vertices)))
        prev = np.sqrt(ctx.residual(xr, z, norms=True)[1][4])
        rates = []
        for _ in range(rho_cycles):
            xr.mul_(1.0 / prev)
            ctx.vcycle(z, xr)
            ctx.gauge(xr)  # the constant pressure is never reduced: project it out
            cur = np.sqrt(ctx.residual(xr, z, norms=True)[1][4])
            rates.append(cur)
            prev = cur
        row[form] = {"ms_per_cycle": round(t_cycle, 3), "rho_last": round(float(rates[-1]), 4),
                     "rho_geo_last10": round(float(np.prod(rates[-10:]) ** 0.1), 4),
                     "n_irregular_rows": int(lay.n_irregular)}
        ctx.close()
    row["speedup_mod_over_sym"] = round(row["sym"]["ms_per_cycle"] / row["mod"]["ms_per_cycle"], 3)
    out["multigrid"].append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
    n *= 2
print(json.dumps(out, indent=1))
