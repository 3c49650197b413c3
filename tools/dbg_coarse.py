import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from oracle import mg
from gpu_util import make_ctx, per_field_rel
ctx, cfg, cls, fcls = make_ctx("cfg1", 16, "mod", kernel_mode=1)
ctx.set_row_n(16)
h = mg.Hierarchy(16, cls, cfg.class_mu, cfg.faces)
l = len(h.levels) - 1
pr = h.levels[l].prob
rng = np.random.default_rng(1)
b = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
xo = h.coarse_solve(b)
xg = ctx.new_vector(l)
ctx.smooth(xg, ctx.import_(b.reshape(4, -1), level=l), 1, level=l)
y = ctx.export(xg, level=l)
print(os.environ.get("STK_DBG_COARSE"), "coarse err", per_field_rel(y, xo))
xo2 = pr.gauge(xo); y2 = pr.gauge(y.reshape(-1))
print("gauged", per_field_rel(y2, xo2))
