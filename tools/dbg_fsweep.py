import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from oracle import mg_mf
from gpu_util import make_ctx, per_field_rel
cfgname, n = sys.argv[1], int(sys.argv[2])
ctx, cfg, cls, fcls = make_ctx(cfgname, n, "mod", kernel_mode=1)
h = mg_mf.MFHierarchy(n, cls, cfg.class_mu, cfg.faces)
pr = h.levels[0].prob
rng = np.random.default_rng(4)
x = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
b = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0) * 1e-3
xs_o = h.uzawa(h.levels[0], x, b)
xg = ctx.import_(x.reshape(4, -1)); bg = ctx.import_(b.reshape(4, -1))
ctx.smooth(xg, bg, 1)
import torch; torch.cuda.synchronize()
err, errs = per_field_rel(ctx.export(xg), xs_o)
print(os.environ.get("STK_FSWEEP"), cfgname, n, "smooth err", err, errs, flush=True)
