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


@pytest.mark.parametrize("cfgname,n", [("cfg1", 16), ("cols", 16), ("cfg2", 16)])
def test_p0_solve_matches_oracle_direct_solution(cfgname, n):
    ctx, cfg, cls, _ = make_ctx(cfgname, n, "mod")
    mu = np.asarray(cfg.class_mu)[cls]
    pr = p1p0.P0Problem(n, mu, cfg.faces, "mod", gamma=1.0)
    V, E = pr.V, pr.E
    rng = np.random.default_rng(6)
    b = np.zeros(3 * V + E)
    b[:3 * V] = np.where(pr.free[:3 * V], rng.uniform(-1, 1, 3 * V), 0.0)
    xo = pr.solve_direct(b)
    b4 = np.zeros((4, V))
    b4[:3] = b[:3 * V].reshape(3, V)
    x, x0, rep = ctx.p0_solve(ctx.import_(b4), torch.zeros(E, dtype=torch.float64, device="cuda"),
                              rtol=1e-11, max_its=400)
    assert rep.rel_res <= 1e-11, (rep.cycles, rep.rel_res)
    xu = ctx.export(x)[:3]
    for a in range(3):
        ref = xo[a * V:(a + 1) * V]
        assert np.linalg.norm(xu[a] - ref) <= 1e-8 * np.linalg.norm(ref)
    ref0 = xo[3 * V:]
    assert np.linalg.norm(x0.cpu().numpy() - ref0) <= 1e-8 * np.linalg.norm(ref0)


def test_p0_solve_couette_flow_reproduces_the_oracle_errors():
    """P:696-713 (mu2/mu1 = 1e-3, interface y = 1/2, exact Dirichlet data lifted into the
    right-hand side by the oracle): the GPU P1-P0 solution equals the oracle's direct
    solution, so it carries the errors of Table couette-results-1e3 (pinned in
    tests/test_oracle_p1p0.py)."""
    import paper_1604_07994_b200 as stk
    for n in (8, 16):
        h = 1.0 / n
        x, y, z = synth._centroids(n, 0, n)
        cls = np.where(y < 0.5, 0, 1).astype(np.uint8).reshape(-1)
        mu = np.array([1.0, 1e-3])
        pr = p1p0.P0Problem(n, mu[cls], synth.ALL_DIRICHLET, "mod", gamma=1.0)
        V, E = pr.V, pr.E
        from oracle import mg
        i, j, k = mg.vertex_coords(n)
        ue = np.stack([0.5 * (1 - (i * h) ** 2), i * h * (j * h - 0.5), 0 * i])
        b = np.zeros(3 * V + E)
        np.add.at(b, pr.vid.reshape(-1), np.repeat(3.0 * mu[cls] * pr.vol / 4.0, 4))
        xd = np.where(pr.free, 0.0, np.concatenate([ue.reshape(-1), np.zeros(E)]))
        beff = np.where(pr.free, b - pr.K @ xd, 0.0)          # lifted rhs (oracle side)
        xo = pr.solve_direct(beff)                             # homogeneous part
        ctx = stk.StokesContext(n, "mod", synth.ALL_DIRICHLET)
        ctx.set_viscosity(cls, mu)
        ctx.assemble()
        b4 = np.zeros((4, V))
        b4[:3] = beff[:3 * V].reshape(3, V)
        xg, x0, rep = ctx.p0_solve(ctx.import_(b4), torch.from_numpy(beff[3 * V:]).cuda(), rtol=1e-11,
                                   max_its=400)
        assert rep.rel_res <= 1e-11, (n, rep.cycles, rep.rel_res)
        xu = ctx.export(xg)[:3].reshape(-1)
        assert np.linalg.norm(xu - xo[:3 * V]) <= 1e-8 * np.linalg.norm(xo[:3 * V])
        assert np.linalg.norm(x0.cpu().numpy() - xo[3 * V:]) <= 1e-8 * np.linalg.norm(xo[3 * V:])
