"""ORACLE (test infrastructure only) — the stabilised P1-P0 scheme of PAPER.md
§3.3-3.4, plain definition with assembled scipy matrices.

* velocity: the P1 space and viscous forms of oracle/fem.py (a_tr), same
  Dirichlet / traction / free-slip elimination;
* pressure: one constant per tetrahedron, element order of synth
  (e = 6 (i + n (j + n k)) + t);
* b(v, q) = -(div v, q): B0[T, (a, v)] = -|T| (grad lambda_m)_a for the local
  vertex m of T at global vertex v;
* c(p, q) = gamma sum_i 1/(2 mu_i) sum_{F interior facet of Omega_i}
  |T1||T2| / (|T1| + |T2|) [p][q]  (eq. stabc): facets between two tets of
  the same viscosity only (no jump penalised across Gamma_12 or on the boundary);
* K0 = [[A, B0^T], [B0, -C0]]  (eq. weakdis / defB), gamma = 1.
* local flux post-process: j_{F;T} = u_h . n_T + Delta j_{F;T} with
  Delta j = gamma / (2 mu |F|) |T||T^F| / (|T| + |T^F|) (p_T - p_{T^F}); element-wise
  sum_F int_F j_{F;T} = 0.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fem
from synth import TRACTION


def _tet_vertices_and_gradients(n):
    """Per element e: global vertex ids (E, 4), |T|, grad lambda (E, 4, 3)."""
    h = 1.0 / n
    E = 6 * n ** 3
    vid = np.empty((E, 4), dtype=np.int64)
    grads = np.empty((E, 4, 3))
    vol = np.empty(E)
    for t in range(6):
        v, g = fem.barycentric_gradients(fem.kuhn_vertices(t) * h)
        vid[t::6] = fem._element_vertex_ids(n, t)
        grads[t::6] = g
        vol[t::6] = v
    return vid, vol, grads


def facets(n):
    """Interior facets as (T1, T2, |F|, unit normal pointing out of T1): every pair of
    tets sharing three vertices (found by sorting the vertex triples of all faces)."""
    vid, vol, grads = _tet_vertices_and_gradients(n)
    E = len(vol)
    tri, owner, opp = [], [], []
    for m in range(4):
        keep = [q for q in range(4) if q != m]
        tri.append(np.sort(vid[:, keep], axis=1))
        owner.append(np.arange(E))
        opp.append(np.full(E, m))
    tri = np.concatenate(tri)
    owner = np.concatenate(owner)
    opp = np.concatenate(opp)
    key = (tri[:, 0] * (1 << 42)) + (tri[:, 1] * (1 << 21)) + tri[:, 2]
    order = np.argsort(key, kind="stable")
    ks = key[order]
    same = np.flatnonzero(ks[1:] == ks[:-1])
    a, b = order[same], order[same + 1]
    T1, T2, m1 = owner[a], owner[b], opp[a]
    # the face opposite local vertex m of T1: outward normal = -grad lambda_m / |grad lambda_m|,
    # |F| = 3 |T| |grad lambda_m|
    g = grads[T1, m1]
    gn = np.linalg.norm(g, axis=1)
    area = 3.0 * vol[T1] * gn
    normal = -g / gn[:, None]
    return T1, T2, area, normal


class P0Problem:
    """The stabilised P1-P0 system on the unit-cube Kuhn grid."""

    def __init__(self, n, elem_mu, faces, form="mod", gamma=1.0):
        self.n, self.gamma = n, gamma
        self.vel = fem.Problem(n, elem_mu, faces, form)      # A, free velocity DoFs
        self.V = self.vel.V
        self.E = 6 * n ** 3
        self.mu = np.asarray(elem_mu, dtype=np.float64).reshape(-1)
        vid, vol, grads = _tet_vertices_and_gradients(n)
        self.vid, self.vol, self.grads = vid, vol, grads
        rows, cols, vals = [], [], []
        for m in range(4):
            for a in range(3):
                rows.append(np.arange(self.E))
                cols.append(vid[:, m] + a * self.V)
                vals.append(-vol * grads[:, m, a])
        self.B = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                               shape=(self.E, 3 * self.V))
        T1, T2, area, normal = facets(n)
        inside = self.mu[T1] == self.mu[T2]           # facets interior to one subdomain
        T1, T2 = T1[inside], T2[inside]
        w = gamma / (2.0 * self.mu[T1]) * vol[T1] * vol[T2] / (vol[T1] + vol[T2])
        self.fT1, self.fT2, self.fw = T1, T2, w
        self.farea, self.fnormal = area[inside], normal[inside]
        C = sp.coo_matrix((np.concatenate([w, w, -w, -w]),
                           (np.concatenate([T1, T2, T1, T2]), np.concatenate([T1, T2, T2, T1]))),
                          shape=(self.E, self.E))
        self.C = C.tocsr()
        self.C.sum_duplicates()
        self.K = sp.bmat([[self.vel.A, self.B.T], [self.B, -self.C]], format="csr")
        self.free = np.concatenate([self.vel.free[:3 * self.V], np.ones(self.E, dtype=bool)])
        self.has_traction = any(f == TRACTION for f in faces)

    def apply(self, x):
        """y = K0 x on the free DoFs (x: 3V velocity then E pressures)."""
        xf = np.where(self.free, x, 0.0)
        return np.where(self.free, self.K @ xf, 0.0)

    def solve_direct(self, b, x_dir=None):
        """K0_FF x_F = b_F - K0_FD x_D; without traction faces the last pressure is
        pinned and the volume-weighted mean pressure removed."""
        free = np.flatnonzero(self.free)
        rhs = b[free].copy()
        if x_dir is not None:
            xd = np.where(self.free, 0.0, x_dir)
            rhs -= (self.K @ xd)[free]
        Kff = self.K[free][:, free].tocsc()
        keep = np.arange(len(free))
        if not self.has_traction:
            keep = keep[:-1]
            Kff = Kff[keep][:, keep]
        sol = np.zeros(len(free))
        sol[keep] = spla.spsolve(Kff.tocsc(), rhs[keep])
        x = np.zeros(3 * self.V + self.E) if x_dir is None else np.where(self.free, 0.0, x_dir)
        x[free] = sol
        if not self.has_traction:
            p = x[3 * self.V:]
            x[3 * self.V:] = p - (self.vol @ p) / self.vol.sum()
        return x

    def facet_fluxes(self, x):
        """per element T and local vertex m, int_F j_{F;T} over the facet F
        opposite m: int_F u_h . n_T (exact for P1: |F| times the mean of u over the facet's
        3 vertices, n_T outward) plus, on facets interior to one subdomain, int_F Delta j
        = gamma/(2 mu) |T||T^F|/(|T|+|T^F|) (p_T - p_{T^F}).  Returns (E, 4)."""
        V = self.V
        u = x[:3 * V].reshape(3, V)
        p = x[3 * V:]
        out = np.zeros((self.E, 4))
        for m in range(4):
            g = self.grads[:, m]
            gn = np.linalg.norm(g, axis=1)
            area = 3.0 * self.vol * gn
            nrm = -g / gn[:, None]
            ubar = np.zeros((self.E, 3))
            for q in range(4):
                if q != m:
                    ubar += u[:, self.vid[:, q]].T / 3.0
            out[:, m] = area * np.sum(ubar * nrm, axis=1)
        # Delta j across interior same-viscosity facets: find the local index of the
        # facet in each tet (the vertex of the tet not on the facet)
        T1, T2, area, normal = facets(self.n)
        same = self.mu[T1] == self.mu[T2]
        for A, Bt in ((T1, T2), (T2, T1)):
            shared = np.zeros(len(A), dtype=np.int64)
            for m in range(4):
                v = self.vid[A, m]
                onB = (self.vid[Bt] == v[:, None]).any(axis=1)
                shared = np.where(~onB, m, shared)
            w = self.gamma / (2.0 * self.mu[A]) * self.vol[A] * self.vol[Bt] / (self.vol[A] + self.vol[Bt])
            np.add.at(out, (A[same], shared[same]), (w * (p[A] - p[Bt]))[same])
        return out

    def facet_flux_balance(self, x):
        """per element, sum over its interior facets of int_F j_{F;T} plus the
        velocity flux through its boundary facets (div theorem: |T| div u_T); returns
        the element-wise balance (0 at solutions of the discrete pressure equation)."""
        V = self.V
        u = x[:3 * V].reshape(3, V)
        p = x[3 * V:]
        # int_{dT} u.n = |T| div u_T
        div = np.zeros(self.E)
        for m in range(4):
            for a in range(3):
                div += self.vol * self.grads[:, m, a] * u[a][self.vid[:, m]]
        bal = div.copy()
        dj = self.fw * (p[self.fT1] - p[self.fT2])       # int_F Delta j_{F;T1}
        np.add.at(bal, self.fT1, dj)
        np.add.at(bal, self.fT2, -dj)
        return bal
