"""-m gpu: the paper's coarse-grid solver through the C
ABI against the oracle (oracle/mg.py, coarse="minres"): one V-cycle with the MINRES
coarse solve (A_sym, corrected right-hand side R25, Jacobi-PCG velocity block, lumped
1/mu mass pressure block, fixed counts R24) on row / element-loop coarse levels, and
a converged solve with it."""
import numpy as np
import pytest

import synth
from oracle import mg
from gpu_util import make_ctx, per_field_rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfgname,n,nc,its,cg,mode", [("cfg1", 16, 4, 20, 4, 1), ("cfg1", 16, 4, 20, 4, 0),
                                                      ("cols", 16, 8, 20, 4, 1), ("cfg2", 32, 8, 12, 3, 1),
                                                      ("cfg5", 32, 16, 10, 2, 1)])
def test_vcycle_with_minres_coarse_solver(cfgname, n, nc, its, cg, mode):
    ctx, cfg, cls, _ = make_ctx(cfgname, n, "mod", kernel_mode=mode, n_coarse=nc)
    ctx.set_coarse_solver("minres", its, cg)
    h = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces, "mod", n_coarse=nc, coarse="minres",
                     minres_its=its, cg_its=cg)
    pr = h.levels[0].prob
    rng = np.random.default_rng(7)
    x = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
    b = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0) * 1e-3
    xg = ctx.import_(x.reshape(4, -1))
    bg = ctx.import_(b.reshape(4, -1))
    ctx.vcycle(bg, xg)
    xo = h.vcycle(b, x)
    err, errs = per_field_rel(ctx.export(xg), xo)
    assert err <= 1e-10, errs


@pytest.mark.parametrize("cfgname,n,nc", [("cfg1", 32, 4), ("cols", 64, 8)])
def test_solve_with_minres_coarse_solver_converges(cfgname, n, nc):
    ctx, cfg, cls, _ = make_ctx(cfgname, n, "mod", n_coarse=nc)
    b = ctx.load_nodal(synth.nodal_forcing(cfg))
    xd, repd = ctx.solve(b, rtol=1e-9, max_cycles=100)
    ctx.set_coarse_solver("minres", 20, 4)
    xm, repm = ctx.solve(b, rtol=1e-9, max_cycles=100)
    assert repm.rel_res <= 1e-9 and repm.cycles <= repd.cycles + 8, (repd.cycles, repm.cycles)
    err, errs = per_field_rel(ctx.export(xm), ctx.export(xd))
    assert err <= 1e-7, errs
