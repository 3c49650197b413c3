"""The process-wide kernel-path switches (environment variables read once per
process) give the same results: each variant runs in its own subprocess and the
outputs are compared.  The default path is pinned to the oracle by
test_gpu_parity.py; these tests pin the alternatives to the default.

* STK_VEL_INPLACE=0: ping-pong velocity colour passes (the repeat pass of the middle
  colour as a copy + the within-colour rows) instead of the in-place passes;
* STK_VEL_INPLACE=0 STK_VEL_REPEAT=0: ping-pong passes with the full repeat pass
  (exact in exact arithmetic);
* STK_LIST_EXPLICIT=0: Gamma rows by the per-thread element loop instead of the
  explicit 4x4-block stencils;
* STK_GJ_GRID=1: coarsest-level inverse by the grid-barrier kernel instead of the
  8-CTA cluster kernel;
* STK_FSWEEP=1: the forward half of the symmetric velocity sweep as ONE fused kernel
  (kernels_sweep.cuh: colour 0 on plane k+1, colour 1 on plane k; list rows around it).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import synth
import paper_1604_07994_b200 as stk
cfg = synth.get_config({cfg!r}, n={n})
cls, fcls = synth.element_classes(cfg)
ctx = stk.StokesContext({n}, {form!r}, cfg.faces, ncolors_u={nc})
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
rng = np.random.default_rng(7)
V = ({n} + 1) ** 3
x = rng.uniform(-1, 1, (4, V))
b = rng.uniform(-1, 1, (4, V)) * 1e-3
xg = ctx.import_(x)
bg = ctx.import_(b)
ctx.smooth(xg, bg, 2)
ctx.vcycle(bg, xg)
np.save({out!r}, ctx.export(xg))
"""


def run_variant(tmp_path, env_extra, cfg, n, form, tag):
    out = str(tmp_path / f"{tag}.npy")
    nc = 4 if form == "sym" else 2
    env = dict(os.environ)
    env.update(env_extra)
    code = SCRIPT.format(root=ROOT, cfg=cfg, n=n, form=form, nc=nc, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def rel(a, b):
    return max(np.linalg.norm(a[f] - b[f]) / max(np.linalg.norm(b[f]), 1e-300) for f in range(4))


@pytest.mark.parametrize("env,cfg,n,form", [
    ({"STK_VEL_INPLACE": "0"}, "cfg2", 128, "mod"),
    ({"STK_VEL_INPLACE": "0", "STK_VEL_REPEAT": "0"}, "cfg5", 64, "grad"),
    ({"STK_VEL_INPLACE": "0", "STK_VEL_REPEAT": "0"}, "cfg3", 128, "mod"),
    ({"STK_LIST_EXPLICIT": "0"}, "cfg2", 128, "mod"),
    ({"STK_LIST_EXPLICIT": "0"}, "cfg2", 64, "sym"),
    ({"STK_GJ_GRID": "1"}, "cfg1", 16, "mod"),
    ({"STK_FSWEEP": "1"}, "cfg2", 128, "mod"),
    ({"STK_FSWEEP": "1"}, "cfg5", 64, "grad"),
    ({"STK_FSWEEP": "1"}, "cfg3", 128, "mod"),
])
def test_switch_matches_default(tmp_path, env, cfg, n, form):
    y_def = run_variant(tmp_path, {}, cfg, n, form, "default")
    y_alt = run_variant(tmp_path, env, cfg, n, form, "alt")
    assert rel(y_alt, y_def) <= 1e-11
