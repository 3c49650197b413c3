"""Debug: V-cycle of the GPU vs oracle for several kernel-path settings."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import synth
from oracle import mg
from gpu_util import make_ctx, per_field_rel
cfgname, n = sys.argv[1], int(sys.argv[2])
for mode, row_n in ((0, 0), (1, 0), (1, 16)):
    ctx, cfg, cls, fcls = make_ctx(cfgname, n, "mod", kernel_mode=mode)
    ctx.set_row_n(row_n)
    h = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces)
    pr = h.levels[0].prob
    rng = np.random.default_rng(3)
    x = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
    b = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0) * 1e-3
    xv_o = h.vcycle(b, x)
    xg = ctx.import_(x.reshape(4, -1))
    bg = ctx.import_(b.reshape(4, -1))
    ctx.vcycle(bg, xg)
    err, errs = per_field_rel(ctx.export(xg), xv_o)
    print(f"{cfgname} n={n} mode={mode} row_n={row_n} row_level={ctx.row_level()} vcycle err {err:.3e} {np.round(errs, 3)}", flush=True)
    # per-level: restrict residual then coarse smoothing on level 1 directly
    for l in range(1, ctx.nlev):
        lev = h.levels[l]
        prl = lev.prob
        xl = np.where(prl.free, rng.uniform(-1, 1, 4 * prl.V), 0.0)
        bl = np.where(prl.free, rng.uniform(-1, 1, 4 * prl.V), 0.0)
        xo = h.uzawa(lev, xl, bl)
        xgl = ctx.import_(xl.reshape(4, -1), level=l)
        ctx.smooth(xgl, ctx.import_(bl.reshape(4, -1), level=l), 1, level=l)
        e1, _ = per_field_rel(ctx.export(xgl, level=l), xo)
        yo = prl.apply(xl)
        yg = ctx.export(ctx.apply(ctx.import_(xl.reshape(4, -1), level=l), level=l), level=l)
        e2, _ = per_field_rel(yg, yo)
        print(f"   level {l} n={lev.n}: smooth err {e1:.2e} apply err {e2:.2e}", flush=True)
