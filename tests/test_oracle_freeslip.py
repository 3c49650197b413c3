"""Pins of the oracle's free-slip boundary (PAPER.md P:104-105:
u.n = 0 and n x sigma(u,p) n = 0 on Gamma_F) against closed forms and
manufactured solutions (-m "not gpu").

* eliminated DoFs: closed-form counts of the face-normal components;
* the viscosity-columns workload of P:772-774 (classes by centroid, the paper's
  forcing of P:719) against its closed-form description;
* K_FF with free slip on all faces: symmetric, kernel = the constant pressure only
  (Korn: no rigid motion is tangential to all six faces);
* manufactured solutions: an isoviscous divergence-free field that is free-slip on
  all six faces, and the two-viscosity MS-1 field, which is free-slip
  on the y and z faces (Dirichlet on x): O(h^2) velocity L2 convergence of the
  consistent forms.  A traction (instead of u.n = 0) face, or the wrong component
  eliminated, breaks the MS-1 field's boundary condition and its rate.
"""
import numpy as np

import synth
from oracle import fem, mg

FS, D = synth.FREESLIP, synth.DIRICHLET


def test_eliminated_mask_counts():
    for n in (2, 4, 7):
        m = synth.eliminated_mask(n, synth.ALL_FREESLIP)
        # component a is eliminated exactly on the two faces of normal e_a
        assert all(m[a].sum() == 2 * (n + 1) ** 2 for a in range(3))
        # corners lose all three components, edges two, face interiors one
        cnt = m.sum(axis=0)
        assert (cnt == 3).sum() == 8
        assert (cnt == 2).sum() == 12 * (n - 1)
        assert (cnt == 1).sum() == 6 * (n - 1) ** 2
    # Dirichlet wins on shared edges: x faces Dirichlet, the rest free slip
    n = 4
    m = synth.eliminated_mask(n, (D, D, FS, FS, FS, FS))
    i, j, k = mg.vertex_coords(n)
    assert m[:, (i == 0) | (i == n)].all()
    assert (m[1] == ((j == 0) | (j == n) | (i == 0) | (i == n))).all()


def test_columns_workload_definition():
    """mu2 = 10 in (0,1/4)^2 x (0,1) u (3/4,1)^2 x (0,1), mu1 = 1 elsewhere;
    free slip; f = (0,0,-cos 2pi x cos 2pi y sin pi z)."""
    cfg = synth.get_config("cols", n=8)
    assert cfg.faces == (FS,) * 6 and cfg.class_mu == (1.0, 10.0)
    cls, _ = synth.element_classes(cfg)
    mu = np.asarray(cfg.class_mu)[cls].reshape(8, 8, 8, 6)
    # each column is 2 x 2 cubes x 8 layers, all 6 tets: volume fraction 2 * (1/4)^2
    assert (mu == 10.0).sum() == 2 * 2 * 2 * 8 * 6
    assert (mu[:, :2, :2] == 10).all() and (mu[:, 6:, 6:] == 10).all()
    assert (mu[:, 2:6] == 1).all() and (mu[:, :, 2:6] == 1).all()
    f = synth.nodal_forcing(cfg)
    i, j, k = mg.vertex_coords(8)
    assert np.allclose(f[:2], 0.0)
    assert np.allclose(f[2], -np.cos(2 * np.pi * i / 8) * np.cos(2 * np.pi * j / 8) * np.sin(np.pi * k / 8))


def test_freeslip_operator_symmetric_with_constant_pressure_kernel():
    n = 4
    cfg = synth.get_config("cols", n=n)
    cls, _ = synth.element_classes(cfg)
    for form in ("mod", "sym", "grad"):
        pr = fem.problem_from_classes(n, cls, cfg.class_mu, cfg.faces, form)
        K = pr.K_free().toarray()
        assert np.abs(K - K.T).max() < 1e-12 * np.abs(K).max()
        s = np.linalg.svd(K, compute_uv=False)
        # exactly one zero singular value: the constant pressure; velocity block
        # nonsingular (no rigid mode satisfies u.n = 0 on all faces of the cube)
        assert s[-1] < 1e-10 * s[0] and s[-2] > 1e-6 * s[0], (form, s[-3:] / s[0])
        free = np.flatnonzero(pr.free)
        const_p = np.where(free >= 3 * pr.V, 1.0, 0.0)
        assert np.abs(K @ const_p).max() < 1e-12 * np.abs(K).max()
        nu = int(np.sum(free < 3 * pr.V))
        Auu = K[:nu, :nu]
        assert np.linalg.eigvalsh(Auu)[0] > 1e-8 * np.abs(Auu).max() or form == "mod"


def _l2_error(pr, x, ue):
    V = pr.V
    e = (x[:3 * V] - ue.reshape(-1)).reshape(3, V)
    return np.sqrt(sum(e[a] @ (pr.M @ e[a]) for a in range(3)))


def _load(pr, n, cls4, fun_by_class):
    """b_u = (phi_i, f)_T with f interpolated per element (consistent mass)."""
    h = 1.0 / n
    b = np.zeros((3, pr.V))
    idx = np.arange(n)
    kk, jj, ii = np.meshgrid(idx, idx, idx, indexing="ij")
    for t in range(6):
        em = fem.element_matrices(t, h, pr.form)
        vid = fem._element_vertex_ids(n, t)
        off = fem.kuhn_vertices(t)
        sub = cls4[..., t].reshape(-1)
        fl = np.zeros((3, n ** 3, 4))
        for m in range(4):
            X = (ii.reshape(-1) + off[m, 0]) * h
            Y = (jj.reshape(-1) + off[m, 1]) * h
            Z = (kk.reshape(-1) + off[m, 2]) * h
            fl[:, :, m] = fun_by_class(sub, X, Y, Z)
        for a in range(3):
            np.add.at(b[a], vid.reshape(-1), (fl[a] @ em["M"].T).reshape(-1))
    return np.where(pr.free, np.concatenate([b.reshape(-1), np.zeros(pr.V)]), 0.0)


def _ms_iso(form, n):
    """u = (sin pi x cos pi y, -cos pi x sin pi y, 0), p = 0, mu = 1: div u = 0, u.n = 0
    and zero tangential traction on all six faces; f = -mu Lap u = 2 pi^2 u."""
    pi = np.pi
    cls = np.zeros(6 * n ** 3, dtype=np.uint8)
    pr = fem.problem_from_classes(n, cls, (1.0,), synth.ALL_FREESLIP, form)

    def u(X, Y, Z):
        return np.stack([np.sin(pi * X) * np.cos(pi * Y), -np.cos(pi * X) * np.sin(pi * Y), 0 * X])

    b = _load(pr, n, cls.reshape(n, n, n, 6), lambda s, X, Y, Z: 2 * pi ** 2 * u(X, Y, Z))
    x = pr.solve_direct(b)
    i, j, k = mg.vertex_coords(n)
    return _l2_error(pr, x, u(i / n, j / n, k / n))


def test_freeslip_isoviscous_manufactured_rates():
    for form in ("mod", "sym", "grad"):
        errs = [_ms_iso(form, n) for n in (4, 8, 16)]
        rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
        assert rates[-1] > 1.8 and errs[-1] < 0.02, (form, errs, rates)


def _ms1_freeslip(form, n):
    """SURVEY App. C MS-1 (mu1 = 10 for x < 1/2, mu2 = 1): u = (a(x) pi cos pi z, 0,
    -a'(x) sin pi z), p = 0.  u_z = 0 and sigma_xz = sigma_yz = 0 on z = 0, 1; u_y = 0 and
    sigma_yx = sigma_yz = 0 on y = 0, 1: free slip there; Dirichlet (the exact u) on x."""
    mu1, mu2 = 10.0, 1.0
    c = (np.pi ** 2 / 2) * (mu2 / mu1 - 1.0)
    pi = np.pi

    def a(x):
        return np.where(x < 0.5, 1 + c * (x - 0.5) ** 2, 1.0)

    def da(x):
        return np.where(x < 0.5, 2 * c * (x - 0.5), 0.0)

    def u(X, Y, Z):
        return np.stack([a(X) * pi * np.cos(pi * Z), 0 * X, -da(X) * np.sin(pi * Z)])

    def f(sub, X, Y, Z):
        f1 = np.stack([pi ** 3 * (16 * mu1 - 8 * mu2 - pi ** 2 * (mu1 - mu2) * (2 * X - 1) ** 2)
                       * np.cos(pi * Z) / 8, 0 * X, pi ** 4 * (mu1 - mu2) * (2 * X - 1) * np.sin(pi * Z) / 2])
        f2 = np.stack([pi ** 3 * mu2 * np.cos(pi * Z), 0 * X, 0 * X])
        return np.where(sub == 0, f1, f2)

    cfg = synth.get_config("cfg1", n=n)
    cls, _ = synth.element_classes(cfg)
    faces = (D, D, FS, FS, FS, FS)
    pr = fem.problem_from_classes(n, cls, (mu1, mu2), faces, form)
    b = _load(pr, n, np.asarray(cls).reshape(n, n, n, 6), f)
    i, j, k = mg.vertex_coords(n)
    ue = u(i / n, j / n, k / n)
    x = pr.solve_direct(b, x_dir=np.concatenate([ue.reshape(-1), np.zeros(pr.V)]))
    return _l2_error(pr, x, ue)


def test_freeslip_interface_manufactured_rates():
    errs = {f: [_ms1_freeslip(f, n) for n in (4, 8, 16)] for f in ("mod", "sym", "grad")}
    for f in ("mod", "sym"):
        rates = np.log2(np.array(errs[f][:-1]) / np.array(errs[f][1:]))
        assert rates[-1] > 1.7 and errs[f][-1] < 0.02, (f, errs[f], rates)
    # the gradient form is inconsistent across the interface
    assert errs["grad"][-1] > 0.2
