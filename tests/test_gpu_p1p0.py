"""-m gpu: the stabilised P1-P0 operator and its
local flux post-process through the C ABI (stk_p0_apply, stk_p0_fluxes)
against the oracle (oracle/p1p0.py), element by element:
velocity rows A u + B0^T p0 and per-tet rows B0 u - C0 p0, within 1e-12 per field, on
Dirichlet (interface), traction-top and free-slip configurations and on a tiled-size
grid (the A block from the TMA stream kernels)."""
import numpy as np
import pytest
import torch

import synth
from oracle import p1p0
from gpu_util import make_ctx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfgname,n,form", [("cfg1", 16, "mod"), ("cfg2", 16, "mod"), ("cols", 16, "mod"),
                                            ("cfg3", 16, "sym"), ("cfg1", 64, "mod"), ("cols", 32, "grad")])
def test_p0_apply_matches_oracle(cfgname, n, form):
    ctx, cfg, cls, _ = make_ctx(cfgname, n, form)
    mu = np.asarray(cfg.class_mu)[cls]
    pr = p1p0.P0Problem(n, mu, cfg.faces, form, gamma=1.0)
    rng = np.random.default_rng(2)
    V, E = pr.V, pr.E
    u = np.where(pr.free[:3 * V], rng.uniform(-1, 1, 3 * V), 0.0)
    p0 = rng.uniform(-1, 1, E)
    yo = pr.apply(np.concatenate([u, p0]))
    x4 = np.zeros((4, V))
    x4[:3] = u.reshape(3, V)
    y, y0 = ctx.p0_apply(ctx.import_(x4), torch.from_numpy(p0).cuda())
    yu = ctx.export(y)[:3]
    for a in range(3):
        ref = yo[a * V:(a + 1) * V]
        assert np.linalg.norm(yu[a] - ref) <= 1e-12 * np.linalg.norm(ref), a
    ref0 = yo[3 * V:]
    got0 = y0.cpu().numpy()
    assert np.linalg.norm(got0 - ref0) <= 1e-12 * np.linalg.norm(ref0)


@pytest.mark.parametrize("cfgname,n", [("cfg1", 16), ("cols", 16), ("cfg2", 32)])
def test_p0_fluxes_match_oracle_and_conserve_on_the_oracle_solution(cfgname, n):
    ctx, cfg, cls, _ = make_ctx(cfgname, n, "mod")
    mu = np.asarray(cfg.class_mu)[cls]
    pr = p1p0.P0Problem(n, mu, cfg.faces, "mod", gamma=1.0)
    V, E = pr.V, pr.E
    rng = np.random.default_rng(4)
    x = np.where(pr.free, rng.uniform(-1, 1, 3 * V + E), 0.0)
    x4 = np.zeros((4, V))
    x4[:3] = x[:3 * V].reshape(3, V)
    fg = ctx.p0_fluxes(ctx.import_(x4), torch.from_numpy(x[3 * V:]).cuda()).cpu().numpy()
    fo = pr.facet_fluxes(x)
    assert np.abs(fg - fo).max() <= 1e-12 * np.abs(fo).max()
    if n <= 16:
        # on the oracle's discrete solution every element conserves mass
        b = np.zeros(3 * V + E)
        b[:3 * V] = np.where(pr.free[:3 * V], rng.uniform(-1, 1, 3 * V), 0.0)
        xs = pr.solve_direct(b)
        x4[:3] = xs[:3 * V].reshape(3, V)
        fs = ctx.p0_fluxes(ctx.import_(x4), torch.from_numpy(xs[3 * V:]).cuda()).cpu().numpy()
        scale = np.abs(fs).max()
        assert np.abs(fs.sum(axis=1)).max() <= 1e-10 * scale
