"""Multi-rank path on one GPU: P contexts of one process on one
device, joined by the loopback exchanger (stk_loopback_create: host rendezvous +
one cudaMemcpyAsync per halo plane / range, one thread per rank, one stream).

The z-slab partition, the halo exchanges, the split coarse levels (own coarse
layers + one layer from the rank below), the agglomeration of the replicated
coarsest levels and the allreduces run exactly as over NCCL on P GPUs.  The apply
must be BITWISE equal to P = 1 (stencils are local, halos are exact copies); the
V-cycle agrees to rounding (the multicolour Gauss-Seidel is independent of the
partition, but the restriction onto / the solve on the replicated coarsest level use
kernels with another summation order than the single-rank row kernels); a solve
agrees up to that and the reduction order of the norms.
"""
import threading

import numpy as np
import pytest

import synth
from gpu_util import make_ctx

pytestmark = pytest.mark.gpu


def run_ranks(P, fn):
    out, err = [None] * P, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append((r, e))

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), "a rank is stuck in a collective"
    assert not err, err
    return out


def make_group(cfgname, n, P, form="mod", krylov=0):
    import paper_1604_07994_b200 as stk
    cfg = synth.get_config(cfgname, n=n)
    grp = stk.LoopbackGroup(P)

    def create(r):
        ctx = stk.StokesContext(n, form, cfg.faces, rank=r, nranks=P, loopback=grp, krylov=krylov)
        cz0, cz1 = ctx.cube_range()
        cls, fcls = synth.element_classes(cfg, cz0, cz1)
        ctx.set_viscosity(cls, cfg.class_mu)
        return ctx, fcls

    ctxs = run_ranks(P, create)
    run_ranks(P, lambda r: ctxs[r][0].assemble())
    return cfg, grp, [c for c, _ in ctxs], [f for _, f in ctxs]


def owned(ctx, arr, n):
    """this rank's owned planes of a canonical (4, (n+1)^3) array"""
    lay = ctx.layout(0)
    N2 = (n + 1) ** 2
    return np.ascontiguousarray(arr[:, lay.z0 * N2:(lay.z0 + lay.nz_local) * N2])


@pytest.mark.parametrize("cfgname,n,P", [("cfg2", 64, 2), ("cfg2", 64, 4), ("cfg3", 64, 4), ("cfg5", 128, 8),
                                        ("cols", 64, 4)])
def test_loopback_apply_bitwise_and_vcycle(cfgname, n, P):
    ctx1, cfg, cls, _ = make_ctx(cfgname, n, "mod")
    x = synth.apply_input(cfg)
    rng = np.random.default_rng(5)
    b = rng.uniform(-1, 1, x.shape) * 1e-3
    y1 = ctx1.export(ctx1.apply(ctx1.import_(x)))
    xv1 = ctx1.import_(x)
    ctx1.vcycle(ctx1.import_(b), xv1)
    v1 = ctx1.export(xv1)
    cfg, grp, ctxs, _ = make_group(cfgname, n, P)
    parts = [c.partition() for c in ctxs]
    assert any(not lv["replicated"] for lv in parts[0][1:]), "no split coarse level exercised"

    def work(r):
        c = ctxs[r]
        y = c.export(c.apply(c.import_(owned(c, x, n))))
        xv = c.import_(owned(c, x, n))
        c.vcycle(c.import_(owned(c, b, n)), xv)
        return y, c.export(xv)

    res = run_ranks(P, work)
    yP = np.concatenate([r[0] for r in res], axis=1)
    vP = np.concatenate([r[1] for r in res], axis=1)
    assert np.array_equal(yP, y1), np.abs(yP - y1).max()
    for fld in range(4):
        assert np.linalg.norm(vP[fld] - v1[fld]) <= 1e-13 * np.linalg.norm(v1[fld])
    # the split coarse levels hold the same element classes / coefficients as P = 1
    for l, lv in enumerate(parts[1]):
        if lv["replicated"] or l == 0:
            continue
        c_r, e_r = ctxs[1].export_classes(l)
        c_1, e_1 = ctx1.export_classes(l)
        m = lv["n"]
        lay = m * m * 6
        np.testing.assert_array_equal(c_r, c_1[lv["cz0"] * lay:lv["cz1"] * lay])
        np.testing.assert_array_equal(e_r, e_1[lv["cz0"] * lay:lv["cz1"] * lay])
    grp.close()


@pytest.mark.parametrize("cfgname,n,P,kry", [("cfg2", 64, 4, 0), ("cfg3", 64, 2, 30), ("cols", 64, 2, 0)])
def test_loopback_solve_matches_single_rank(cfgname, n, P, kry):
    ctx1, cfg, cls, fcls = make_ctx(cfgname, n, "mod", krylov=kry)
    if cfg.forcing == "nodal":
        f = synth.nodal_forcing(cfg)
        b1 = ctx1.load_nodal(f)
    else:
        b1 = ctx1.load_element(fcls, cfg.force_table)
    x1, rep1 = ctx1.solve(b1, rtol=1e-10, max_cycles=200)
    s1 = ctx1.export(x1)
    cfg, grp, ctxs, fcl = make_group(cfgname, n, P, krylov=kry)

    def work(r):
        c = ctxs[r]
        if cfg.forcing == "nodal":
            bb = c.load_nodal(owned(c, f, n)[:3])
        else:
            bb = c.load_element(fcl[r], cfg.force_table)
        xs, rep = c.solve(bb, rtol=1e-10, max_cycles=200)
        return c.export(xs), rep.cycles, rep.rel_res

    res = run_ranks(P, work)
    sP = np.concatenate([r[0] for r in res], axis=1)
    assert all(r[2] <= 1e-10 for r in res)
    assert abs(res[0][1] - rep1.cycles) <= 1
    for fld in range(4):
        assert np.linalg.norm(sP[fld] - s1[fld]) <= 1e-9 * np.linalg.norm(s1[fld])
    grp.close()
