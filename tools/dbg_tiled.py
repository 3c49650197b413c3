import sys
sys.path.insert(0, ".")
import numpy as np
import synth
from oracle import capi
import paper_1604_07994_b200 as stk
sys.path.insert(0, "tests")
from gpu_util import make_ctx, per_field_rel
n = 64
ctx, cfg, cls, _ = make_ctx("cfg4", n, "mod", kernel_mode=1)
x = synth.apply_input(cfg)
y_o = capi.apply_slab(n, "mod", 1 / 12, cfg.faces, cls, cfg.class_mu, x).reshape(4, -1)
y_g = ctx.export(ctx.apply(ctx.import_(x)))
print("apply err", per_field_rel(y_g, y_o))
