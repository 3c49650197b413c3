"""ORACLE (test infrastructure only) — the same multigrid as oracle.mg, with the
level operators applied by the plain C element loop (oracle/c/oracle.c) instead
of assembled scipy matrices, so that smoother / V-cycle parity can be checked
on grids (n = 64, 128) where the tiled GPU kernels run.  The algorithm is the
one of oracle.mg.Hierarchy (inherited); only the matrix products differ.
"""
from __future__ import annotations

import numpy as np

from synth import TRACTION, dirichlet_vertex_mask, eliminated_mask
from . import capi, fem, mg


class _Op:
    def __init__(self, fn, T=None):
        self._fn = fn
        self._T = T

    def __matmul__(self, v):
        return self._fn(v)

    @property
    def T(self):
        return self._T


class MFProblem:
    """Matrix-free level: products by the C element loop (blocks A, B^T, B, C)."""

    def __init__(self, n, mu_a, imu_c, faces, form="mod", delta=1.0 / 12.0):
        self.n, self.V = n, (n + 1) ** 3
        self.h = 1.0 / n
        self.mu_a = np.ascontiguousarray(mu_a, dtype=np.float64)
        self.imu_c = np.ascontiguousarray(imu_c, dtype=np.float64)
        self.faces, self.form, self.delta = tuple(faces), form, delta
        self.dir_v = dirichlet_vertex_mask(n, self.faces)
        self.free = np.concatenate([~eliminated_mask(n, self.faces).reshape(-1), np.ones(self.V, dtype=bool)])
        self.has_traction = any(f == TRACTION for f in self.faces)
        V = self.V

        def ap(vec, blocks):
            return capi.apply_slab(n, form, delta, self.faces, None, None, vec, blocks=blocks,
                                   mu_a=self.mu_a, imu_c=self.imu_c)

        def A(u):
            return ap(np.concatenate([u, np.zeros(V)]), 1)[:3 * V]

        def BT(p):
            return ap(np.concatenate([np.zeros(3 * V), p]), 2)[:3 * V]

        def B(u):
            return ap(np.concatenate([u, np.zeros(V)]), 4)[3 * V:]

        def C(p):
            return -ap(np.concatenate([np.zeros(3 * V), p]), 8)[3 * V:]

        self.A = _Op(A)
        self.B = _Op(B, _Op(BT))
        self.C = _Op(C)
        self._ap = ap
        dA, dC = capi.diagonals(n, form, delta, self.faces, None, None, mu_a=self.mu_a, imu_c=self.imu_c)
        self.diagA, self.diagC = dA, dC
        # gauge weights w_j = sum_T |T| / (4 mu_T)
        w = np.zeros(V)
        imu = self.imu_c.reshape(n, n, n, 6)
        for t in range(6):
            vid = fem._element_vertex_ids(n, t)
            np.add.at(w, vid.reshape(-1), np.repeat((self.h ** 3 / 6) * imu[..., t].reshape(-1) / 4.0, 4))
        self.gauge_w = w

    def apply(self, x):
        return np.where(self.free, self._ap(np.where(self.free, x.reshape(-1), 0.0), 15), 0.0)

    gauge = fem.Problem.gauge


class MFLevel:
    def __init__(self, n, cls, mu_a, imu_c, faces, form, delta):
        self.n = n
        self.cls = np.asarray(cls, dtype=np.uint8)
        self.mu_a, self.imu_c = mu_a, imu_c
        if n <= 16:
            self.prob = fem.Problem(n, mu_a, faces, form, delta, elem_imu_c=imu_c)
            self.diagA = self.prob.A.diagonal()
            self.diagC = self.prob.C.diagonal()
        else:
            self.prob = MFProblem(n, mu_a, imu_c, faces, form, delta)
            self.diagA, self.diagC = self.prob.diagA, self.prob.diagC
        i, j, k = mg.vertex_coords(n)
        self.parity = i + j + k
        self.free_u = self.prob.free[:3 * self.prob.V]


class MFHierarchy(mg.Hierarchy):
    def __init__(self, n, cls, class_mu, faces, form="mod", delta=1.0 / 12.0,
                 n_coarse=4, nu_pre=3, nu_post=3, nu_inc=2, omega=0.3, ncolors_u=2,
                 coarse="direct", minres_its=20, cg_its=4, coarse_mu="arith"):
        self.levels, self.P = [], []
        c = np.asarray(cls, dtype=np.uint8)
        mu_a = np.asarray(class_mu, dtype=np.float64)[c]
        imu_c = 1.0 / mu_a
        m = n
        while True:
            self.levels.append(MFLevel(m, c, mu_a, imu_c, faces, form, delta))
            if m <= n_coarse:
                break
            self.P.append(mg.prolongation(m // 2))
            mu_a, imu_c = mg.coarse_viscosity(m, mu_a, imu_c, coarse_mu)
            c = mg.coarse_classes(m, c)
            m //= 2
        self.nu_pre, self.nu_post, self.nu_inc = nu_pre, nu_post, nu_inc
        self.omega = omega
        self.ncolors_u = ncolors_u
        self.coarse, self.minres_its, self.cg_its = coarse, minres_its, cg_its
        self.faces, self.delta = tuple(faces), delta
        self._coarse_setup()
