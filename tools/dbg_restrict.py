import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from oracle import mg
from gpu_util import make_ctx
ctx, cfg, cls, fcls = make_ctx("cfg1", 32, "mod", kernel_mode=1)
ctx.set_row_n(16)
h = mg.Hierarchy(32, cls, cfg.class_mu, cfg.faces)
rng = np.random.default_rng(1)
l = 2
pr = h.levels[l].prob; pc = h.levels[l + 1].prob
ro = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
P = h.P[l]
bc = np.where(pc.free, np.concatenate([P.T @ ro.reshape(4, -1)[f] for f in range(4)]), 0.0).reshape(4, -1)
rv = ctx.import_(ro.reshape(4, -1), level=l)
lay = ctx.layout(l)
print("layout", lay.n, lay.pitch_x, lay.pitch_y, lay.field_stride, lay.vec_len)
bcg = ctx.export(ctx.restrict(rv, fine_level=l), level=l + 1)
d = np.abs(bcg - bc)
nc = pc.n + 1
for f in range(4):
    bad = np.flatnonzero(d[f] > 1e-12)
    print("field", f, "bad", len(bad), "of", nc ** 3, [(v % nc, (v // nc) % nc, v // nc ** 2) for v in bad[:12]])
    if len(bad):
        v = bad[0]; print("   gpu", bcg[f, v], "oracle", bc[f, v])
