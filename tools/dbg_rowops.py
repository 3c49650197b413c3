import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from oracle import mg, fem
from gpu_util import make_ctx, per_field_rel
ctx, cfg, cls, fcls = make_ctx("cfg1", 32, "mod", kernel_mode=1)
ctx.set_row_n(16)
h = mg.Hierarchy(32, cls, cfg.class_mu, cfg.faces)
rng = np.random.default_rng(1)
for l in (1, 2):
    pr = h.levels[l].prob
    x = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
    b = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
    ro = b - pr.apply(x)
    rg = ctx.export(ctx.residual(ctx.import_(x.reshape(4, -1), level=l), ctx.import_(b.reshape(4, -1), level=l), level=l), level=l)
    print("level", l, "residual", per_field_rel(rg, ro)[0], flush=True)
    if l + 1 < len(h.levels):
        P = h.P[l]
        pc = h.levels[l + 1].prob
        bc = np.where(pc.free, np.concatenate([P.T @ ro.reshape(4, -1)[f] for f in range(4)]), 0.0)
        bcg = ctx.export(ctx.restrict(ctx.import_(ro.reshape(4, -1), level=l), fine_level=l), level=l + 1)
        print("level", l, "restrict", per_field_rel(bcg, bc)[0], flush=True)
        xc = np.where(pc.free, rng.uniform(-1, 1, 4 * pc.V), 0.0)
        xf = np.where(pr.free, (x + np.concatenate([P @ xc.reshape(4, -1)[f] for f in range(4)])), 0.0)
        xg = ctx.import_(x.reshape(4, -1), level=l)
        ctx.prolong_add(ctx.import_(xc.reshape(4, -1), level=l + 1), xg, coarse_level=l + 1)
        print("level", l, "prolong", per_field_rel(ctx.export(xg, level=l), xf)[0], flush=True)
