"""Shared helpers for the -m gpu parity tests (test harness only)."""
import numpy as np

import synth


def per_field_rel(a, b, V=None):
    """max over the 4 fields of ||a_f - b_f|| / ||b_f|| (fields of length V)."""
    a = np.asarray(a).reshape(4, -1)
    b = np.asarray(b).reshape(4, -1)
    out = []
    for f in range(4):
        nb = np.linalg.norm(b[f])
        out.append(np.linalg.norm(a[f] - b[f]) / (nb if nb > 0 else 1.0))
    return max(out), out


def make_ctx(cfgname, n, form="mod", kernel_mode=None, **kw):
    import paper_1604_07994_b200 as stk
    cfg = synth.get_config(cfgname, n=n)
    cls, fcls = synth.element_classes(cfg)
    ctx = stk.StokesContext(n, form, cfg.faces, **kw)
    if kernel_mode is not None:
        ctx.set_kernel_mode(kernel_mode)
    ctx.set_viscosity(cls, cfg.class_mu)
    ctx.assemble()
    return ctx, cfg, cls, fcls


def rhs_oracle_and_gpu(ctx, cfg, cls, fcls, prob):
    """(b_oracle, b_gpu_vector) for the config's forcing."""
    if cfg.forcing == "nodal":
        f = synth.nodal_forcing(cfg)
        return prob.load_nodal(f), ctx.load_nodal(f)
    fe = np.asarray(cfg.force_table)[fcls]
    return prob.load_element(fe), ctx.load_element(fcls, cfg.force_table)
