"""Pins of the oracle against what PAPER.md and the mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of them re-types the oracle's own
formulas: they use closed forms, invariants, an independent surface-integral
construction of eq. (decouple), the manufactured solution of SURVEY App. C,
brute-force loops on tiny inputs, or the direct solution.
"""
import itertools

import numpy as np
import pytest
import scipy.sparse as sp

import synth
from oracle import fem, mg


def _cfg1_problem(n=8, form="mod", faces=synth.ALL_DIRICHLET, mu=(10.0, 1.0), delta=1 / 12):
    cfg = synth.get_config("cfg1", n=n)
    cls, _ = synth.element_classes(cfg)
    return fem.problem_from_classes(n, cls, mu, faces, form, delta), cls


def _position_field(n):
    i, j, k = mg.vertex_coords(n)
    return np.stack([i, j, k]).astype(float) / n


# -- P:1309 DoF convention ------------------------------------------------------
def test_dof_count_matches_paper_coarse_grid():
    # "level L=2 with 19 652 DoF for the coarse grid": 4 (n+1)^3 at n = 16
    assert synth.get_config("cfg1").dofs == 19652
    # L = 7, 8: 5.4e8 and 4.3e9 DoF
    assert round(synth.get_config("cfg4").dofs / 1e8, 1) == 5.4
    assert round(synth.get_config("cfg5").dofs / 1e9, 1) == 4.3


# -- barycentric gradients: defining property of the hat functions ---------------
@pytest.mark.parametrize("t", range(6))
def test_barycentric_gradients_define_hat_functions(t):
    v = fem.kuhn_vertices(t) * 0.25
    vol, g = fem.barycentric_gradients(v)
    assert vol == pytest.approx(0.25 ** 3 / 6)
    for i in range(4):
        for j in range(4):
            # lambda_i(a_j) - lambda_i(a_0) = g_i . (a_j - a_0) = delta_ij - delta_i0
            assert g[i] @ (v[j] - v[0]) == pytest.approx(float(i == j) - float(i == 0), abs=1e-12)
    # every cube is split into 6 tets of equal volume covering it
    assert 6 * vol == pytest.approx(0.25 ** 3)


# -- a_tr(x,x) = -3 sum mu_i|Omega_i|, a_dev(x,x) = 0 --------------------
@pytest.mark.parametrize("form,factor", [("grad", 3.0), ("sym", 6.0), ("mod", -3.0), ("dev", 0.0)])
def test_position_field_closed_forms(form, factor):
    n = 8
    pr, _ = _cfg1_problem(n, form)
    x = _position_field(n).reshape(-1)
    Mmu = 10.0 * 0.5 + 1.0 * 0.5        # sum_i mu_i |Omega_i| for cfg1
    val = x @ (pr.A @ x)
    assert val == pytest.approx(factor * Mmu, abs=1e-10)


def test_divergence_of_position_field():
    # b(x, q) = -(div x, q) = -3 int q; all rows including the boundary
    n = 6
    pr, _ = _cfg1_problem(n)
    x = _position_field(n).reshape(-1)
    intphi = pr.M @ np.ones(pr.V)
    np.testing.assert_allclose(pr.B @ x, -3.0 * intphi, atol=1e-14)
    # interior vertices: int phi_i = h^3
    i, j, k = mg.vertex_coords(n)
    inner = (i > 0) & (i < n) & (j > 0) & (j < n) & (k > 0) & (k < n)
    np.testing.assert_allclose(intphi[inner], (1 / n) ** 3, rtol=1e-13)


def test_rigid_modes_and_constants():
    n = 5
    pr, _ = _cfg1_problem(n, "mod")
    V = pr.V
    for a in range(3):                     # constant velocity: grad u = 0
        e = np.zeros(3 * V)
        e[a * V:(a + 1) * V] = 1.0
        assert np.abs(pr.A @ e).max() < 1e-12
        assert np.abs(pr.B @ e).max() < 1e-14
    assert np.abs(pr.C @ np.ones(V)).max() < 1e-14
    # pressure constant mode of the constrained system when Gamma_F is empty
    x = np.zeros(4 * V)
    x[3 * V:] = 1.0
    assert np.abs(pr.apply(x)).max() < 1e-14
    # ... and not with a traction face (Gamma_F fixes the pressure)
    prt, _ = _cfg1_problem(n, "mod", faces=synth.TOP_TRACTION)
    assert np.abs(prt.apply(x)).max() > 1e-3


@pytest.mark.parametrize("form", ["mod", "sym", "grad", "dev"])
def test_symmetry(form):
    pr, _ = _cfg1_problem(6, form, faces=synth.TOP_TRACTION)
    assert abs(pr.A - pr.A.T).max() < 1e-13
    assert abs(pr.C - pr.C.T).max() < 1e-18
    assert abs(pr.K - pr.K.T).max() < 1e-13


def test_forms_relations():
    # a_tr = a_sym - (mu div, div) = a_dev - (1/3)(mu div, div)   (d = 3)
    n = 4
    ps = {f: _cfg1_problem(n, f)[0] for f in ("mod", "sym", "dev", "grad")}
    pr, cls = ps["mod"], _cfg1_problem(n)[1]
    # (mu div u, div v) assembled independently from divergence of each hat function
    D = ps["sym"].A - ps["mod"].A
    np.testing.assert_allclose((ps["dev"].A - D / 3.0 - pr.A).toarray(), 0.0, atol=1e-13)
    # D is positive semi-definite and equals mu * (div)^T (div) per element:
    # u^T D u = sum_T mu_T |T| (div_T u)^2 for random u
    rng = np.random.default_rng(1)
    u = rng.standard_normal(3 * pr.V)
    mu = np.asarray((10.0, 1.0))[cls].reshape(n, n, n, 6)
    h = 1 / n
    U = u.reshape(3, n + 1, n + 1, n + 1)          # [a][k][j][i]
    tot = 0.0
    for k, j, i, t in itertools.product(range(n), range(n), range(n), range(6)):
        verts = fem.kuhn_vertices(t).astype(int) + np.array([i, j, k])
        # divergence of the linear interpolant: fit u_a = c + g.x through 4 vertices
        X = np.hstack([np.ones((4, 1)), verts * h])
        div = 0.0
        for a in range(3):
            vals = np.array([U[a, vz, vy, vx] for vx, vy, vz in verts])
            coef = np.linalg.solve(X, vals)
            div += coef[1 + a]
        tot += mu[k, j, i, t] * (h ** 3 / 6) * div ** 2
    assert u @ (D @ u) == pytest.approx(tot, rel=1e-12)


# -- BASELINE north_star: mu1 = mu2, Dirichlet only => A_tr = A_grad on free DoFs ----
def test_modified_equals_gradient_isoviscous_dirichlet():
    n = 6
    pm, _ = _cfg1_problem(n, "mod", mu=(3.0, 3.0))
    pg, _ = _cfg1_problem(n, "grad", mu=(3.0, 3.0))
    f = np.flatnonzero(pm.free[:3 * pm.V])
    d = (pm.A[f][:, f] - pg.A[f][:, f]).toarray()
    assert np.abs(d).max() < 1e-13
    # but not with a jump or with a traction face
    pj, _ = _cfg1_problem(n, "mod")
    pgj, _ = _cfg1_problem(n, "grad")
    assert np.abs((pj.A[f][:, f] - pgj.A[f][:, f]).toarray()).max() > 1e-2
    pt, _ = _cfg1_problem(n, "mod", faces=synth.TOP_TRACTION, mu=(3.0, 3.0))
    pgt, _ = _cfg1_problem(n, "grad", faces=synth.TOP_TRACTION, mu=(3.0, 3.0))
    ft = np.flatnonzero(pt.free[:3 * pt.V])
    assert np.abs((pt.A[ft][:, ft] - pgt.A[ft][:, ft]).toarray()).max() > 1e-2


# -- Lemma rotation-identity ---------------------------------------------
R3 = [np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0]]),
      np.array([[0, 0, 1], [0, 0, 0], [-1, 0, 0]]),
      np.array([[0, -1, 0], [1, 0, 0], [0, 0, 0]])]


def test_rotation_identity():
    rng = np.random.default_rng(0)
    T = rng.standard_normal((3, 3))
    lhs = T - np.trace(T) * np.eye(3)
    rhs = sum(R @ T.T @ R for R in R3)
    np.testing.assert_allclose(lhs, rhs, atol=1e-14)
    x = rng.standard_normal(3)
    for j in range(3):
        np.testing.assert_allclose(R3[j] @ x, np.cross(np.eye(3)[j], x), atol=1e-15)


# -- eq. (decouple): a_tr = (mu grad, grad) - [mu] sum_j (d_tj u, R^j v)_G12
#                                  - mu sum_j (d_tj u, R^j v)_GF   — by surface quadrature
def _surface_form(n, faces_pred, normal, weight_of_face):
    """Assemble sum_j (d_{t_j} u, R^j v)_F * weight over mesh facets F selected by
    faces_pred, t_j = R^j n.  Independent of the oracle: facets enumerated from the
    tet faces, tangential gradients from the facet geometry."""
    V = (n + 1) ** 3
    h = 1.0 / n
    N1 = n + 1
    seen = {}
    for k, j, i, t in itertools.product(range(n), range(n), range(n), range(6)):
        verts = fem.kuhn_vertices(t).astype(int) + np.array([i, j, k])
        for drop in range(4):
            tri = tuple(sorted(tuple(v) for m, v in enumerate(verts) if m != drop))
            if faces_pred(np.array(tri) * h) and tri not in seen:
                seen[tri] = (k, j, i, t)
    rows, cols, vals = [], [], []
    eps = np.zeros((3, 3, 3))
    for a, b, c in itertools.permutations(range(3)):
        eps[a, b, c] = np.linalg.det(np.eye(3)[[a, b, c]])
    tvec = [np.cross(np.eye(3)[j], normal) for j in range(3)]
    for tri, owner in seen.items():
        P = np.array(tri, dtype=float) * h
        e1, e2 = P[1] - P[0], P[2] - P[0]
        area = 0.5 * np.linalg.norm(np.cross(e1, e2))
        Msys = np.stack([e1, e2, normal])
        gid = [tv[0] + N1 * (tv[1] + N1 * tv[2]) for tv in tri]
        w = weight_of_face(owner)
        for m in range(3):
            psi = np.zeros(3)
            psi[m] = 1.0
            gm = np.linalg.solve(Msys, np.array([psi[1] - psi[0], psi[2] - psi[0], 0.0]))
            for l in range(3):
                for a in range(3):
                    for b in range(3):
                        s = sum((gm @ tvec[jj]) * eps[b, jj, a] for jj in range(3))
                        if s != 0.0:
                            rows.append(a * V + gid[l])
                            cols.append(b * V + gid[m])
                            vals.append(w * s * area / 3.0)
    return sp.csr_matrix((vals, (rows, cols)), shape=(3 * V, 3 * V))


def test_decouple_equivalence_interface_and_traction():
    n = 4
    mu = (10.0, 1.0)
    pm, cls = _cfg1_problem(n, "mod", faces=synth.TOP_TRACTION, mu=mu)
    pg, _ = _cfg1_problem(n, "grad", faces=synth.TOP_TRACTION, mu=mu)
    cls4 = np.asarray(cls).reshape(n, n, n, 6)
    S12 = _surface_form(n, lambda P: np.allclose(P[:, 0], 0.5), np.array([1.0, 0, 0]),
                        lambda o: mu[0] - mu[1])                      # [mu] = mu1 - mu2, n = n_1
    SF = _surface_form(n, lambda P: np.allclose(P[:, 2], 1.0), np.array([0, 0, 1.0]),
                       lambda o: mu[cls4[o]])                          # mu of the adjacent tet
    f = np.flatnonzero(pm.free[:3 * pm.V])
    lhs = pm.A[f][:, f].toarray()
    rhs = (pg.A - S12 - SF)[f][:, f].toarray()
    assert np.abs(lhs - rhs).max() < 1e-13 * np.abs(lhs).max()


def test_cross_part_only_on_interface_rows():
    # the full stencil is needed only at Gamma_12 and Gamma_F rows;
    # X = A_tr - A_grad lives on interface rows x interface columns, off the
    # diagonal component blocks, antisymmetric in the components.
    n = 8
    pm, cls = _cfg1_problem(n, "mod", faces=synth.TOP_TRACTION, mu=(1e3, 1.0))
    pg, _ = _cfg1_problem(n, "grad", faces=synth.TOP_TRACTION, mu=(1e3, 1.0))
    V = pm.V
    X = (pm.A - pg.A).tocoo()
    f = pm.free[:3 * V]
    keep = f[X.row] & f[X.col] & (np.abs(X.data) > 1e-13 * abs(pm.A).max())
    r, c, d = X.row[keep], X.col[keep], X.data[keep]
    i, j, k = mg.vertex_coords(n)
    iface = (2 * i == n) | (k == n)
    assert iface[r % V].all() and iface[c % V].all()
    assert ((r // V) != (c // V)).all()
    Xf = sp.csr_matrix((d, (r, c)), shape=(3 * V, 3 * V)).toarray()
    for a, b in itertools.permutations(range(3), 2):
        blk_ab = Xf[a * V:(a + 1) * V, b * V:(b + 1) * V]
        blk_ba = Xf[b * V:(b + 1) * V, a * V:(a + 1) * V]
        np.testing.assert_allclose(blk_ab, -blk_ba, atol=1e-13 * abs(pm.A).max())
        assert np.abs(np.diag(blk_ab)).max() < 1e-13 * abs(pm.A).max()


# -- transfers: nodal interpolation reproduces linear functions ------------------
def test_prolongation_reproduces_linears():
    nc = 4
    P = mg.prolongation(nc)
    xc = _position_field(nc)
    xf = _position_field(2 * nc)
    rng = np.random.default_rng(3)
    c = rng.standard_normal(4)
    lin_c = c[0] + c[1:] @ xc
    lin_f = c[0] + c[1:] @ xf
    np.testing.assert_allclose(P @ lin_c, lin_f, atol=1e-14)
    np.testing.assert_allclose(P @ np.ones(P.shape[1]), 1.0, atol=1e-15)
    # entries are 1 (coinciding vertices) or 1/2 (edge midpoints) only
    assert set(np.round(P.data, 12)) <= {0.5, 1.0}


def test_coarse_classes_of_resolved_interface_equal_rediscretisation():
    # a resolved interface (cfg1 plane x = 1/2) gives pure coarse classes that equal
    # the direct classification of the coarse grid (no MIXED tet)
    cf = synth.get_config("cfg1", n=16)
    cc = synth.get_config("cfg1", n=8)
    cls_f, _ = synth.element_classes(cf)
    cls_c, _ = synth.element_classes(cc)
    got = mg.coarse_classes(16, cls_f)
    np.testing.assert_array_equal(got, cls_c)
    mu_a, imu_c = mg.coarse_viscosity(16, np.asarray(cf.class_mu)[cls_f], 1.0 / np.asarray(cf.class_mu)[cls_f])
    np.testing.assert_allclose(mu_a, np.asarray(cf.class_mu)[cls_c], rtol=1e-15)
    np.testing.assert_allclose(imu_c, 1.0 / np.asarray(cf.class_mu)[cls_c], rtol=1e-15)


def _bey_children_brute(nf, K, J, I, T):
    """Fine tets whose centroid lies strictly inside coarse tet (K,J,I,T)."""
    verts = (fem.kuhn_vertices(T) + np.array([I, J, K])) * 2.0
    Xc = np.hstack([np.ones((4, 1)), verts])
    out = []
    for k, j, i, t in itertools.product(range(nf), range(nf), range(nf), range(6)):
        cen = (fem.kuhn_vertices(t) + np.array([i, j, k])).mean(axis=0)
        lam = np.linalg.solve(Xc.T, np.concatenate([[1.0], cen]))
        if (lam > 1e-12).all():
            out.append(((k * nf + j) * nf + i) * 6 + t)
    return out


def test_coarse_viscosity_and_class_brute_force():
    # reading R15 by brute force: every coarse tet has exactly 8 Bey children; mu_A is
    # their arithmetic mean, 1/mu_C the mean of their 1/mu, the class is shared or MIXED
    rng = np.random.default_rng(5)
    nf = 4
    cls = rng.integers(0, 3, size=6 * nf ** 3).astype(np.uint8)
    cls[:6 * nf * nf] = 1                  # a layer of pure coarse tets too
    mu = np.array([1.0, 7.0, 3.0])
    mu_a, imu_c = mg.coarse_viscosity(nf, mu[cls], 1.0 / mu[cls])
    mu_h, imu_h = mg.coarse_viscosity(nf, mu[cls], 1.0 / mu[cls], "harmonic")
    cc = mg.coarse_classes(nf, cls)
    seen_mixed = seen_pure = False
    for K, J, I, T in itertools.product(range(2), range(2), range(2), range(6)):
        ch = _bey_children_brute(nf, K, J, I, T)
        assert len(ch) == 8
        e = ((K * 2 + J) * 2 + I) * 6 + T
        assert mu_a[e] == pytest.approx(np.mean(mu[cls[ch]]), rel=1e-15)
        assert imu_c[e] == pytest.approx(np.mean(1.0 / mu[cls[ch]]), rel=1e-15)
        # stk_config.coarse_mu = 2: harmonic mean for A, the same 1/mu_C
        assert mu_h[e] == pytest.approx(8.0 / np.sum(1.0 / mu[cls[ch]]), rel=1e-15)
        assert imu_h[e] == imu_c[e]
        if len(set(cls[ch])) == 1:
            assert cc[e] == cls[ch[0]]
            seen_pure = True
        else:
            assert cc[e] == mg.MIXED
            seen_mixed = True
    assert seen_mixed and seen_pure


@pytest.mark.parametrize("form", ["mod", "sym", "grad"])
def test_coarse_operators_are_galerkin_products(form):
    # R15 pinned against the Galerkin products of the nested P1 spaces (P:573-574,
    # R = P^T): with mu_A the arithmetic mean of the children, the coarse
    # A equals P^T A_f P; B_c = P^T B_f P exactly; with 1/mu_C the mean of 1/mu the
    # coarse C equals 4 P^T C_f P (C carries h_l^2, R1, and h_c = 2 h_f).
    nf, nc = 8, 4
    rng = np.random.default_rng(11)
    mu_f = np.array([1.0, 1e3, 30.0])[rng.integers(0, 3, size=6 * nf ** 3)]
    faces = synth.TOP_TRACTION
    pf = fem.Problem(nf, mu_f, faces, form)
    mu_a, imu_c = mg.coarse_viscosity(nf, mu_f, 1.0 / mu_f)
    pc = fem.Problem(nc, mu_a, faces, form, elem_imu_c=imu_c)
    P = mg.prolongation(nc)
    P3 = sp.block_diag([P] * 3).tocsr()
    fu = sp.diags(pf.free[:3 * pf.V].astype(float))
    cu = pc.free[:3 * pc.V]
    Ag = (P3.T @ fu @ pf.A @ fu @ P3).toarray()[np.ix_(cu, cu)]
    Ac = pc.A.toarray()[np.ix_(cu, cu)]
    assert np.abs(Ag - Ac).max() <= 1e-12 * np.abs(Ac).max()
    Bg = (P.T @ pf.B @ fu @ P3).toarray()[:, cu]
    np.testing.assert_allclose(Bg, pc.B.toarray()[:, cu], atol=1e-14 * np.abs(Bg).max())
    Cg = 4.0 * (P.T @ pf.C @ P).toarray()
    np.testing.assert_allclose(Cg, pc.C.toarray(), atol=1e-12 * np.abs(Cg).max())
    # the gauge weights keep int_Omega 1/mu (the coarse weight of a tet is |T_c| times
    # the mean of 1/mu over its children)
    assert pc.gauge_w.sum() == pytest.approx(pf.gauge_w.sum(), rel=1e-13)


# -- Q = {q : int mu^-1 q = 0}; gauge weights w_j = int phi_j / mu -------------
def test_gauge_weights_closed_forms():
    n = 8
    pr, cls = _cfg1_problem(n, "mod", mu=(10.0, 1.0))
    # sum_j w_j = int_Omega 1/mu = |Omega_1|/mu_1 + |Omega_2|/mu_2 (plane x = 1/2)
    assert pr.gauge_w.sum() == pytest.approx(0.5 / 10.0 + 0.5 / 1.0, rel=1e-13)
    # an isoviscous interior vertex: int phi_j = h^3 (mu = 10 left, 1 right)
    i, j, k = mg.vertex_coords(n)
    inner = (i > 0) & (j > 0) & (k > 0) & (i < n) & (j < n) & (k < n)
    left, right = inner & (2 * i < n), inner & (2 * i > n)
    np.testing.assert_allclose(pr.gauge_w[left], (1 / n) ** 3 / 10.0, rtol=1e-13)
    np.testing.assert_allclose(pr.gauge_w[right], (1 / n) ** 3 / 1.0, rtol=1e-13)
    # a constant pressure is gauged to 0; a gauged field has zero weighted mean
    x = np.zeros(4 * pr.V)
    x[3 * pr.V:] = 3.7
    assert np.abs(pr.gauge(x)[3 * pr.V:]).max() < 1e-13
    rng = np.random.default_rng(2)
    x[3 * pr.V:] = rng.standard_normal(pr.V)
    assert abs(pr.gauge_w @ pr.gauge(x)[3 * pr.V:]) < 1e-14


# -- consistent mass (load_nodal) against the App. A.2 closed-form stencil -----------
def test_load_nodal_matches_mass_stencil():
    n = 6
    pr, _ = _cfg1_problem(n, "mod")
    h = 1.0 / n
    N1 = n + 1
    rng = np.random.default_rng(4)
    f = rng.standard_normal((3, pr.V))
    b = pr.load_nodal(f).reshape(4, pr.V)
    # interior row of M: h^3 [2/5 centre; 1/20 at +-e_s and +-(1,1,1); 1/30 at
    # +-(1,1,0), +-(1,0,1), +-(0,1,1)]
    sten = {(0, 0, 0): 2 / 5}
    for d in [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)]:
        sten[d] = sten[tuple(-c for c in d)] = 1 / 20
    for d in [(1, 1, 0), (1, 0, 1), (0, 1, 1)]:
        sten[d] = sten[tuple(-c for c in d)] = 1 / 30
    assert sum(sten.values()) == pytest.approx(1.0)
    for (i, j, k) in [(1, 1, 1), (3, 2, 4), (5, 5, 5), (2, 4, 1)]:
        v = i + N1 * (j + N1 * k)
        for a in range(3):
            want = h ** 3 * sum(w * f[a, (i + d[0]) + N1 * ((j + d[1]) + N1 * (k + d[2]))]
                                for d, w in sten.items())
            assert b[a, v] == pytest.approx(want, rel=1e-12)
    assert np.abs(b[3]).max() == 0.0                       # b_p = 0
    dmask = synth.dirichlet_vertex_mask(n, synth.ALL_DIRICHLET)
    assert np.abs(b[:3, dmask]).max() == 0.0


def test_load_nodal_elementwise_equals_assembled_mass():
    n = 5
    pr, _ = _cfg1_problem(n, "mod", faces=synth.TOP_TRACTION)
    f = np.random.default_rng(12).standard_normal((3, pr.V))
    np.testing.assert_allclose(fem.load_nodal_elementwise(n, synth.TOP_TRACTION, f), pr.load_nodal(f),
                               rtol=1e-13, atol=1e-17)


def test_load_element_brute_force_and_total():
    # element-constant f: b_{i,a} = sum_{T ni i} f_{T,a} |T| / 4 (R10).  Brute force
    # on one tet, and sum_i b_{i,a} = int f_a when no vertex is constrained.
    n = 3
    faces = (synth.TRACTION,) * 6                           # no constrained velocity row
    pr = fem.Problem(n, np.ones(6 * n ** 3), faces, "mod")
    rng = np.random.default_rng(6)
    E = 6 * n ** 3
    fe = rng.standard_normal((E, 3))
    b = pr.load_element(fe).reshape(4, pr.V)
    vol = (1 / n) ** 3 / 6
    np.testing.assert_allclose(b[:3].sum(axis=1), fe.sum(axis=0) * vol, rtol=1e-12)
    one = np.zeros((E, 3))
    e = 6 * (1 + n * (2 + n * 0)) + 4                         # cube (1,2,0), tet 4
    one[e] = (1.0, -2.0, 0.5)
    b1 = pr.load_element(one).reshape(4, pr.V)
    verts = fem.kuhn_vertices(4).astype(int) + np.array([1, 2, 0])
    ids = [vx + (n + 1) * (vy + (n + 1) * vz) for vx, vy, vz in verts]
    want = np.zeros((3, pr.V))
    for v in ids:
        want[:, v] = np.array([1.0, -2.0, 0.5]) * vol / 4
    np.testing.assert_allclose(b1[:3], want, atol=1e-17)


# -- smoother: Jacobi-within-colour == Gauss-Seidel for rows without same-colour coupling
def test_colour_pass_equals_sequential_gauss_seidel_on_7pt_rows():
    n = 4
    pg, cls = _cfg1_problem(n, "grad")
    h = mg.Hierarchy(n, cls, (10.0, 1.0), synth.ALL_DIRICHLET, form="grad", n_coarse=4)
    lev = h.levels[0]
    V = pg.V
    rng = np.random.default_rng(7)
    u0 = np.where(lev.free_u, rng.standard_normal(3 * V), 0.0)
    rhs = rng.standard_normal(3 * V)
    A = pg.A.tocsr()
    # sequential GS, vertex by vertex: colour 0 then colour 1 then 1 then 0
    u = u0.copy()
    order = []
    for c in (0, 1, 1, 0):
        order += [r for r in range(3 * V) if lev.parity[r % V] % 2 == c and lev.free_u[r]]
    for r in order:
        s = rhs[r]
        for idx in range(A.indptr[r], A.indptr[r + 1]):
            cidx = A.indices[idx]
            if cidx != r:
                s -= A.data[idx] * u[cidx]
        u[r] = s / A[r, r]
    # oracle's vectorised colour sweep (pressure fixed at 0, rhs given through f)
    x = np.concatenate([u0, np.zeros(V)])
    b = np.concatenate([rhs, np.zeros(V)])
    hx = h
    hx.omega = 0.0
    out = hx.uzawa(lev, x, b)
    np.testing.assert_allclose(out[:3 * V], u, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("faces", [synth.ALL_DIRICHLET, synth.TOP_TRACTION])
def test_pressure_sweep_equals_sequential_forward_gauss_seidel(faces):
    # S^ of P:1243 ("forward variant of the Gauss-Seidel method applied to ... C,
    # omega = 0.3"), reading R11: delta = one forward Gauss-Seidel sweep on
    # C delta = r_p from 0 in red-black order, p += omega delta.  Checked against a
    # row-by-row sequential sweep written here; a Jacobi sweep would fail it.
    n = 4
    cfg = synth.get_config("cfg1", n=n)
    cls, _ = synth.element_classes(cfg)
    h = mg.Hierarchy(n, cls, (10.0, 1.0), faces, n_coarse=4)
    lev = h.levels[0]
    pr = lev.prob
    V = pr.V
    rng = np.random.default_rng(8)
    x = np.where(pr.free, rng.standard_normal(4 * V), 0.0)
    b = np.where(pr.free, rng.standard_normal(4 * V), 0.0)
    out = h.uzawa(lev, x, b)
    u1 = out[:3 * V]                          # velocity half: pinned by the 7-pt test above
    rp = pr.B @ u1 - pr.C @ x[3 * V:] - b[3 * V:]
    C = pr.C.tocsr()
    par = lev.parity % 2
    # C couples only vertices of different parity (7-point), so red-black = GS
    Cc = C.tocoo()
    off = (Cc.row != Cc.col) & (np.abs(Cc.data) > 1e-14 * np.abs(Cc.data).max())
    assert (par[Cc.row[off]] != par[Cc.col[off]]).all()
    d = np.zeros(V)
    for colour in (0, 1):
        for r in [v for v in range(V) if par[v] == colour]:
            s_ = rp[r]
            for idx in range(C.indptr[r], C.indptr[r + 1]):
                if C.indices[idx] != r:
                    s_ -= C.data[idx] * d[C.indices[idx]]
            d[r] = s_ / C[r, r]
    want = x[3 * V:] + 0.3 * d
    np.testing.assert_allclose(out[3 * V:], want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
    jac = x[3 * V:] + 0.3 * rp / C.diagonal()
    assert np.abs(jac - want).max() > 1e-3 * np.abs(want).max()


def test_exact_solution_is_smoother_and_vcycle_fixed_point():
    n = 8
    cfg = synth.get_config("cfg1", n=n)
    cls, _ = synth.element_classes(cfg)
    h = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces)
    pr = h.levels[0].prob
    b = pr.load_nodal(synth.nodal_forcing(cfg))
    xs = pr.solve_direct(b)
    np.testing.assert_allclose(h.uzawa(h.levels[0], xs, b), xs, atol=1e-11)
    np.testing.assert_allclose(pr.gauge(h.vcycle(b, xs)), xs, atol=1e-10)


def test_coarse_solve_consistent_rhs():
    n = 8
    cfg = synth.get_config("cfg1", n=n)
    cls, _ = synth.element_classes(cfg)
    h = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces, n_coarse=8)
    pr = h.levels[-1].prob
    rng = np.random.default_rng(9)
    xt = pr.gauge(np.where(pr.free, rng.standard_normal(4 * pr.V), 0.0))
    b = pr.apply(xt)
    np.testing.assert_allclose(h.coarse_solve(b), xt, atol=1e-9)


@pytest.mark.parametrize("cfgname,form", [("cfg1", "mod"), ("cfg1", "sym"), ("cfg2", "mod")])
def test_multigrid_reaches_direct_solution(cfgname, form):
    n = 16
    cfg = synth.get_config(cfgname, n=n)
    cls, _ = synth.element_classes(cfg)
    h = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces, form=form,
                     ncolors_u=4 if form == "sym" else 2)
    pr = h.levels[0].prob
    b = pr.load_nodal(synth.nodal_forcing(cfg))
    xd = pr.solve_direct(b)
    x, hist = h.solve(b, rtol=1e-12, max_cycles=60)
    assert hist[-1] <= 1e-12
    rho = (hist[-1] / hist[3]) ** (1 / (len(hist) - 4))
    assert rho < 0.6
    for fld in range(4):
        s = slice(fld * pr.V, (fld + 1) * pr.V)
        assert np.linalg.norm(x[s] - xd[s]) <= 1e-8 * np.linalg.norm(xd[s])


@pytest.mark.parametrize("cfgname", ["cfg3", "cfg5"])
def test_krylov_multigrid_reaches_direct_solution_high_contrast(cfgname):
    # unresolved 1e3-1e4 inclusions (BASELINE cfg3, cfg5): GMRES preconditioned by the
    # V_var cycle with the R15 coarse viscosities reaches the unique discrete solution
    n = 16
    cfg = synth.get_config(cfgname, n=n)
    cls, fcls = synth.element_classes(cfg)
    h = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces)
    pr = h.levels[0].prob
    b = pr.load_element(fem.element_force(n, fcls, cfg.force_table))
    xd = pr.gauge(pr.solve_direct(b))
    x, rel = h.solve_krylov(b, rtol=1e-11)
    assert rel <= 1e-10
    for fld in range(4):
        s = slice(fld * pr.V, (fld + 1) * pr.V)
        assert np.linalg.norm(x[s] - xd[s]) <= 1e-8 * np.linalg.norm(xd[s])


# -- SURVEY App. C manufactured solution MS-1: O(h^2) velocity L2 for mod/sym,
#    no convergence for grad ("convergence to a wrong solution") ----------------
def _ms1(form, n):
    mu1, mu2 = 10.0, 1.0
    c = (np.pi ** 2 / 2) * (mu2 / mu1 - 1.0)
    pi = np.pi

    def a(x):
        return np.where(x < 0.5, 1 + c * (x - 0.5) ** 2, 1.0)

    def da(x):
        return np.where(x < 0.5, 2 * c * (x - 0.5), 0.0)

    def u_exact(x, y, z):
        return np.stack([a(x) * pi * np.cos(pi * z), 0 * x, -da(x) * np.sin(pi * z)])

    def f1(x, y, z):
        return np.stack([pi ** 3 * (16 * mu1 - 8 * mu2 - pi ** 2 * (mu1 - mu2) * (2 * x - 1) ** 2)
                         * np.cos(pi * z) / 8, 0 * x, pi ** 4 * (mu1 - mu2) * (2 * x - 1) * np.sin(pi * z) / 2])

    def f2(x, y, z):
        return np.stack([pi ** 3 * mu2 * np.cos(pi * z), 0 * x, 0 * x])

    cfg = synth.get_config("cfg1", n=n)
    cls, _ = synth.element_classes(cfg)
    pr = fem.problem_from_classes(n, cls, (mu1, mu2), synth.ALL_DIRICHLET, form)
    h = 1.0 / n
    V = pr.V
    cls4 = np.asarray(cls).reshape(n, n, n, 6)
    b = np.zeros((3, V))
    for t in range(6):
        em = fem.element_matrices(t, h, form)
        vid = fem._element_vertex_ids(n, t)
        off = fem.kuhn_vertices(t)
        idx = np.arange(n)
        kk, jj, ii = np.meshgrid(idx, idx, idx, indexing="ij")
        sub = cls4[..., t].reshape(-1)
        fl = np.zeros((3, n ** 3, 4))
        for m in range(4):
            X = (ii.reshape(-1) + off[m, 0]) * h
            Y = (jj.reshape(-1) + off[m, 1]) * h
            Z = (kk.reshape(-1) + off[m, 2]) * h
            fl[:, :, m] = np.where(sub == 0, f1(X, Y, Z), f2(X, Y, Z))
        for a_ in range(3):
            loc = fl[a_] @ em["M"].T
            np.add.at(b[a_], vid.reshape(-1), loc.reshape(-1))
    bb = np.concatenate([b.reshape(-1), np.zeros(V)])
    bb = np.where(pr.free, bb, 0.0)
    i, j, k = mg.vertex_coords(n)
    ue = u_exact(i * h, j * h, k * h)
    xd = np.concatenate([ue.reshape(-1), np.zeros(V)])
    x = pr.solve_direct(bb, x_dir=xd)
    e = (x[:3 * V] - ue.reshape(-1)).reshape(3, V)
    return np.sqrt(sum(e[a_] @ (pr.M @ e[a_]) for a_ in range(3)))


def test_manufactured_solution_rates():
    errs = {f: [_ms1(f, n) for n in (4, 8, 16)] for f in ("mod", "sym", "grad")}
    for f in ("mod", "sym"):
        rates = np.log2(np.array(errs[f][:-1]) / np.array(errs[f][1:]))
        assert rates[-1] > 1.7, (f, errs[f], rates)
        assert errs[f][-1] < 0.02
    # gradient form converges to a wrong solution: error does not decrease
    assert errs["grad"][-1] > 0.2 and errs["grad"][-1] > 0.8 * errs["grad"][0]
    # modified and strain-based errors are near-identical (consistency)
    assert abs(errs["mod"][-1] - errs["sym"][-1]) < 0.25 * errs["sym"][-1]
