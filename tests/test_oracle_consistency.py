"""The three oracle realisations agree (-m "not gpu"): scipy assembly (pinned in
test_oracle_pins.py), the C element loop, and the matrix-free multigrid."""
import numpy as np
import pytest

import synth
from oracle import capi, fem, mg, mg_mf


@pytest.mark.parametrize("cfgname,form", [("cfg1", "mod"), ("cfg2", "sym"), ("cfg2", "grad"),
                                          ("cfg5", "mod"), ("cfg3", "mod")])
def test_c_element_loop_equals_assembly(cfgname, form):
    n = 8
    cfg = synth.get_config(cfgname, n=n)
    cls, _ = synth.element_classes(cfg)
    pr = fem.problem_from_classes(n, cls, cfg.class_mu, cfg.faces, form)
    x = synth.apply_input(cfg).reshape(-1)
    y0 = pr.apply(x)
    y1 = capi.apply_slab(n, form, 1 / 12, cfg.faces, cls, cfg.class_mu, x)
    assert np.abs(y0 - y1).max() <= 1e-14 * np.abs(y0).max()
    y2 = capi.apply_slab(n, form, 1 / 12, cfg.faces, cls, cfg.class_mu, x, 3, 6)
    sl = slice(3 * (n + 1) ** 2, 6 * (n + 1) ** 2)
    assert np.abs((y0 - y2).reshape(4, -1)[:, sl]).max() <= 1e-14 * np.abs(y0).max()
    rows = capi.apply_rows(n, form, 1 / 12, cfg.faces, cls, cfg.class_mu, x, np.arange(pr.V))
    assert np.abs(rows.T.reshape(-1) - y0).max() <= 1e-14 * np.abs(y0).max()
    dA, dC = capi.diagonals(n, form, 1 / 12, cfg.faces, cls, cfg.class_mu)
    np.testing.assert_allclose(dA, pr.A.diagonal(), rtol=1e-14)
    np.testing.assert_allclose(dC, pr.C.diagonal(), rtol=1e-14)


def test_matrix_free_multigrid_equals_assembled():
    n = 32
    cfg = synth.get_config("cfg2", n=n)
    cls, _ = synth.element_classes(cfg)
    h = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces)
    hm = mg_mf.MFHierarchy(n, cls, cfg.class_mu, cfg.faces)
    pr = h.levels[0].prob
    rng = np.random.default_rng(0)
    x = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0)
    b = np.where(pr.free, rng.uniform(-1, 1, 4 * pr.V), 0.0) * 1e-3
    a, c = h.uzawa(h.levels[0], x, b), hm.uzawa(hm.levels[0], x, b)
    assert np.abs(a - c).max() <= 1e-14 * np.abs(a).max()
    a, c = h.vcycle(b, x), hm.vcycle(b, x)
    assert np.abs(a - c).max() <= 1e-13 * np.abs(a).max()
