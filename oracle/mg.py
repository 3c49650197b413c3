"""ORACLE (test infrastructure only) — all-at-once Uzawa V_var multigrid.

Written from PAPER.md §5 with assembled scipy matrices:

* Uzawa smoothing step, eq. (Uzawa_smooth)
      u <- u + A^^-1 (f - A u - B^T p)
      p <- p + S^^-1 (B u - C p - g)
  A^ : symmetric coloured Gauss-Seidel on A ("symmetric hybrid parallel variant of
       a row-wise red-black colored Gauss-Seidel").  Reading R12
       (DESIGN.md): colours c(v) = (i+j+k) mod nc, colour passes 0..nc-1 then
       nc-1..0; inside one colour pass every row of that colour is relaxed from
       the vector at the start of the pass (Jacobi within a colour — the
       "hybrid").  For rows without same-colour couplings this is exact GS.
  S^ : "forward variant of the Gauss-Seidel method applied to ... C, with
       omega = 0.3".  Reading R11: delta = one forward red-black GS sweep
       on C delta = r from delta = 0, then p += omega * delta.
* V_var cycle: nu_l = nu + nu_inc * l smoothing steps before and after
  on level l (l = 0 finest; reading R13).
* "Standard restriction and prolongation": P = coarse P1 basis evaluated
  at fine vertices (plain definition of the nodal interpolation), R = P^T.
* Coarse operators rediscretised per level (h_l = 1/n_l) with per-element coarse
  viscosities (reading R15): for a coarse tet T_c with Bey children
  T_1..T_8 (the fine tets whose centroids lie in T_c)
      mu_A(T_c)    = (1/8) sum_q mu_A(T_q)        arithmetic mean  (viscous block A)
      1/mu_C(T_c)  = (1/8) sum_q 1/mu_C(T_q)      harmonic mean    (weight of C, gauge)
  The first makes the rediscretised coarse A equal to the Galerkin product
  P^T A_f P of the nested P1 spaces (R = P^T, "standard" transfers P:1243); the
  second gives C the Galerkin viscosity weight at the coarse h_l.  A coarse tet's
  class is the common class of its children, or MIXED.
* Coarsest level: exact solve ("a direct coarse grid solver ... is not
  problematic") of the free-DoF system; without a traction face the pressure
  constant is fixed by the Lagrange row w^T p = 0 (reading R9/R16).
  Or (coarse="minres") the paper's Krylov coarse solver, P:1245-1298:
  the coarse system is re-discretised with the strain form A_sym (same coarse
  viscosities), the momentum right-hand side is corrected by B^T M_L^-1 r2, and the
  system [[A_sym, B^T], [B, -C]] is solved by MINRES preconditioned with
  blockdiag(A^, M_L): A^^-1 = Jacobi-preconditioned CG on A_sym.  Reading R25
  (DESIGN.md): M_L = the lumped mass weighted by 1/mu (diag int phi_i / mu, = the
  paper's lumped mass for mu = 1), and the correction is r1 + B^T M_L^-1 r2 -- with
  b(v,q) = -(div v, q) and a_sym = a_tr + (mu div, div) this is the
  sign that makes the two coarse systems agree (B z ~ -M_L div z); the printed
  "r1 - B^T M^-1 r2" moves the A_sym solution away from the A_tr one (pinned
  in tests/test_oracle_coarse_minres.py).  The paper's stopping criteria are not printed ("selected such that the
  multigrid convergence rates do not deteriorate"): fixed iteration counts here,
  stopping early only when gamma_{j+1} <= 1e-14 gamma_1 (reading R24), MINRES from zero.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fem import Problem, barycentric_gradients, kuhn_vertices
from synth import PERMS


def vertex_coords(n: int):
    idx = np.arange(n + 1)
    k, j, i = np.meshgrid(idx, idx, idx, indexing="ij")
    return i.reshape(-1), j.reshape(-1), k.reshape(-1)


def _locate(points: np.ndarray, nc: int, strict: bool):
    """For points in coarse-grid units, the coarse (cube, type, barycentric) containing
    them: barycentric coordinates w.r.t. each of the 6 Kuhn tets of the cube, first
    tet with all coordinates >= 0 (strict: > 0)."""
    cube = np.minimum(np.floor(points).astype(np.int64), nc - 1)
    local = points - cube
    found_t = np.full(len(points), -1)
    lam_out = np.zeros((len(points), 4))
    for t in range(6):
        _, g = barycentric_gradients(kuhn_vertices(t))
        a0 = kuhn_vertices(t)[0]
        # lambda_i(q) = lambda_i(a0) + g_i . (q - a0);  lambda_i(a0) = delta_i0
        lam = (local - a0) @ g.T
        lam[:, 0] += 1.0
        ok = (lam > 1e-12).all(axis=1) if strict else (lam > -1e-12).all(axis=1)
        take = ok & (found_t < 0)
        found_t[take] = t
        lam_out[take] = lam[take]
    assert (found_t >= 0).all()
    return cube, found_t, lam_out


def prolongation(nc: int) -> sp.csr_matrix:
    """P[f, c] = phi_c(x_f): coarse P1 hat functions at the fine vertices (nf = 2 nc)."""
    nf = 2 * nc
    i, j, k = vertex_coords(nf)
    pts = np.stack([i, j, k], axis=1) / 2.0
    cube, t, lam = _locate(pts, nc, strict=False)
    rows, cols, vals = [], [], []
    N1 = nc + 1
    for m in range(4):
        off = np.stack([kuhn_vertices(tt)[m] for tt in range(6)]).astype(np.int64)[t]
        cv = cube + off
        cid = cv[:, 0] + N1 * (cv[:, 1] + N1 * cv[:, 2])
        keep = np.abs(lam[:, m]) > 1e-14
        rows.append(np.arange(len(pts))[keep])
        cols.append(cid[keep])
        vals.append(lam[keep, m])
    P = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=((nf + 1) ** 3, N1 ** 3))
    P.sum_duplicates()
    return P


MIXED = 0xFE   # class of a coarse tet whose children do not share one class


def child_parent(nf: int) -> np.ndarray:
    """For every fine tet (flattened [k][j][i][t]) the flattened index of the coarse
    tet (grid nf/2) that contains its centroid: the Bey parent."""
    nc = nf // 2
    idx = np.arange(nf)
    kk, jj, ii = np.meshgrid(idx, idx, idx, indexing="ij")
    out = np.empty((nf, nf, nf, 6), dtype=np.int64)
    for t in range(6):
        cen = kuhn_vertices(t).mean(axis=0)
        pts = np.stack([ii.reshape(-1) + cen[0], jj.reshape(-1) + cen[1],
                        kk.reshape(-1) + cen[2]], axis=1) / 2.0
        cube, tc, _ = _locate(pts, nc, strict=True)
        out[..., t] = (6 * (cube[:, 0] + nc * (cube[:, 1] + nc * cube[:, 2])) + tc).reshape(nf, nf, nf)
    out = out.reshape(-1)
    assert (np.bincount(out, minlength=6 * nc ** 3) == 8).all()
    return out


def coarse_viscosity(nf: int, mu_a: np.ndarray, imu_c: np.ndarray, mode: str = "arith"):
    """Coarse per-element (mu_A, 1/mu_C): means over the 8 Bey children (reading R15);
    mode "harmonic": mu_A = 8 / sum 1/mu_A (stk_config.coarse_mu = 2)."""
    par = child_parent(nf)
    E = 6 * (nf // 2) ** 3
    if mode == "harmonic":
        mu_c = 8.0 / np.bincount(par, weights=1.0 / np.asarray(mu_a, dtype=np.float64).reshape(-1), minlength=E)
    else:
        mu_c = np.bincount(par, weights=np.asarray(mu_a, dtype=np.float64).reshape(-1), minlength=E) / 8.0
    imu_cc = np.bincount(par, weights=np.asarray(imu_c, dtype=np.float64).reshape(-1), minlength=E) / 8.0
    return mu_c, imu_cc


def coarse_classes(nf: int, cls_f: np.ndarray) -> np.ndarray:
    """Coarse class: the class shared by all 8 Bey children, else MIXED."""
    par = child_parent(nf)
    E = 6 * (nf // 2) ** 3
    c = np.asarray(cls_f, dtype=np.int64).reshape(-1)
    lo = np.full(E, 1 << 20)
    hi = np.full(E, -1)
    np.minimum.at(lo, par, c)
    np.maximum.at(hi, par, c)
    return np.where(lo == hi, lo, MIXED).astype(np.uint8)


class Level:
    def __init__(self, n, cls, mu_a, imu_c, faces, form, delta):
        self.n = n
        self.cls = np.asarray(cls, dtype=np.uint8)
        self.mu_a, self.imu_c = mu_a, imu_c
        self.prob = Problem(n, mu_a, faces, form, delta, elem_imu_c=imu_c)
        i, j, k = vertex_coords(n)
        self.parity = (i + j + k)
        V = self.prob.V
        self.diagA = self.prob.A.diagonal()
        self.diagC = self.prob.C.diagonal()
        self.free_u = self.prob.free[:3 * V]


class Hierarchy:
    def __init__(self, n, cls, class_mu, faces, form="mod", delta=1.0 / 12.0,
                 n_coarse=4, nu_pre=3, nu_post=3, nu_inc=2, omega=0.3, ncolors_u=2,
                 coarse="direct", minres_its=20, cg_its=4, coarse_mu="arith"):
        self.levels = []
        self.P = []
        c = np.asarray(cls, dtype=np.uint8)
        mu_a = np.asarray(class_mu, dtype=np.float64)[c]
        imu_c = 1.0 / mu_a
        m = n
        while True:
            self.levels.append(Level(m, c, mu_a, imu_c, faces, form, delta))
            if m <= n_coarse:
                break
            assert m % 2 == 0
            self.P.append(prolongation(m // 2))
            mu_a, imu_c = coarse_viscosity(m, mu_a, imu_c, coarse_mu)
            c = coarse_classes(m, c)
            m //= 2
        self.nu_pre, self.nu_post, self.nu_inc = nu_pre, nu_post, nu_inc
        self.omega = omega
        self.ncolors_u = ncolors_u
        self.coarse, self.minres_its, self.cg_its = coarse, minres_its, cg_its
        self.faces, self.delta = tuple(faces), delta
        self._coarse_setup()

    # -- smoother ----------------------------------------------------------
    def uzawa(self, lev: Level, x: np.ndarray, b: np.ndarray) -> np.ndarray:
        pr = lev.prob
        V = pr.V
        x = x.copy()
        u, p = x[:3 * V], x[3 * V:]
        f, g = b[:3 * V], b[3 * V:]
        rhs = f - pr.B.T @ p
        nc = self.ncolors_u
        col_u = np.tile(lev.parity % nc, 3)
        for c in list(range(nc)) + list(reversed(range(nc))):
            r = rhs - pr.A @ u
            sel = (col_u == c) & lev.free_u
            u[sel] += r[sel] / lev.diagA[sel]
        rp = pr.B @ u - pr.C @ p - g
        d = np.zeros(V)
        col_p = lev.parity % 2
        for c in range(2):
            s = rp - pr.C @ d
            sel = col_p == c
            d[sel] += s[sel] / lev.diagC[sel]
        p += self.omega * d
        return x

    # -- coarse solve ------------------------------------------------------
    def _coarse_setup(self):
        if self.coarse == "minres":
            self._minres_setup()
            return
        lev = self.levels[-1]
        pr = lev.prob
        free = np.flatnonzero(pr.free)
        Kff = pr.K[free][:, free].toarray()
        if not pr.has_traction:
            w = np.concatenate([np.zeros(3 * pr.V), pr.gauge_w])[free]
            N = len(free)
            Kaug = np.zeros((N + 1, N + 1))
            Kaug[:N, :N] = Kff
            Kaug[:N, N] = w
            Kaug[N, :N] = w
            self.G = np.linalg.inv(Kaug)[:N, :N]
        else:
            self.G = np.linalg.inv(Kff)
        self.coarse_free = free

    def coarse_solve(self, b):
        if self.coarse == "minres":
            return self.coarse_solve_minres(b)
        x = np.zeros_like(b)
        x[self.coarse_free] = self.G @ b[self.coarse_free]
        return x

    # -- the paper's coarse solver ----------------------------
    def _minres_setup(self):
        lev = self.levels[-1]
        self.psym = Problem(lev.n, lev.mu_a, self.faces, "sym", self.delta, elem_imu_c=lev.imu_c)
        V = self.psym.V
        self.ml = self.psym.gauge_w.copy()           # lumped 1/mu-weighted mass (R25)
        self.dsym = self.psym.A.diagonal()                            # Jacobi for A_sym
        self.fu = self.psym.free[:3 * V]

    def jacobi_pcg(self, r):
        """A^^-1 r: cg_its steps of Jacobi-preconditioned CG on A_sym (free velocity
        DoFs) from zero."""
        A, fu = self.psym.A, self.fu
        dinv = np.where(fu, 1.0 / np.where(fu, self.dsym, 1.0), 0.0)
        x = np.zeros_like(r)
        r = np.where(fu, r, 0.0)
        z = dinv * r
        p = z.copy()
        rz = r @ z
        for k in range(self.cg_its):
            if rz == 0.0:
                break
            Ap = np.where(fu, A @ p, 0.0)
            alpha = rz / (p @ Ap)
            x += alpha * p
            r = r - alpha * Ap
            if k + 1 == self.cg_its:
                break
            z = dinv * r
            rz_new = r @ z
            p = z + (rz_new / rz) * p
            rz = rz_new
        return x

    def coarse_solve_minres(self, b):
        """RHS correction r1 + B^T M_L^-1 r2 (R25), then preconditioned MINRES on
        [[A_sym, B^T], [B, -C]] (Elman-Silvester-Wathen preconditioned MINRES, x0 = 0)
        with the preconditioner blockdiag(A^, M_L), minres_its iterations."""
        pr = self.psym
        V = pr.V
        free = pr.free

        def K(x):
            return np.where(free, pr.K @ np.where(free, x, 0.0), 0.0)

        def Pinv(v):
            return np.concatenate([self.jacobi_pcg(v[:3 * V]), v[3 * V:] / self.ml])

        r = np.where(free, b, 0.0).copy()
        r[:3 * V] += pr.B.T @ (r[3 * V:] / self.ml)               # r1 + B^T M_L^-1 r2 (R25)
        r = np.where(free, r, 0.0)
        x = np.zeros_like(r)
        v_old = np.zeros_like(r)
        v = r.copy()
        z = Pinv(v)
        gamma = np.sqrt(max(z @ v, 0.0))
        if gamma == 0.0:
            return x
        gamma_old, gamma0 = 1.0, gamma
        eta = gamma
        s_old = s = 0.0
        c_old = c = 1.0
        w_old = np.zeros_like(r)
        w = np.zeros_like(r)
        for _ in range(self.minres_its):
            z = z / gamma
            Kz = K(z)
            delta = Kz @ z
            v_new = Kz - (delta / gamma) * v - (gamma / gamma_old) * v_old
            z_new = Pinv(v_new)
            gamma_new = np.sqrt(max(z_new @ v_new, 0.0))
            a0 = c * delta - c_old * s * gamma
            a1 = np.sqrt(a0 * a0 + gamma_new * gamma_new)
            a2 = s * delta + c_old * c * gamma
            a3 = s_old * gamma
            c_old, s_old = c, s
            c, s = a0 / a1, gamma_new / a1
            w_new = (z - a3 * w_old - a2 * w) / a1
            x = x + c * eta * w_new
            eta = -s * eta
            v_old, v = v, v_new
            w_old, w = w, w_new
            z = z_new
            gamma_old, gamma = gamma, gamma_new
            if gamma <= 1e-14 * gamma0:       # converged to rounding: stop (R24)
                break
        return x

    # -- cycle -------------------------------------------------------------
    def vcycle(self, b, x, l=0):
        lev = self.levels[l]
        if l == len(self.levels) - 1:
            return self.coarse_solve(b)
        for _ in range(self.nu_pre + self.nu_inc * l):
            x = self.uzawa(lev, x, b)
        r = b - lev.prob.apply(x)
        P = self.P[l]
        Vc = self.levels[l + 1].prob.V
        bc = np.concatenate([P.T @ r.reshape(4, -1)[f] for f in range(4)])
        bc = np.where(self.levels[l + 1].prob.free, bc, 0.0)
        xc = self.vcycle(bc, np.zeros(4 * Vc), l + 1)
        x = x + np.concatenate([P @ xc.reshape(4, -1)[f] for f in range(4)])
        x = np.where(lev.prob.free, x, 0.0)
        for _ in range(self.nu_post + self.nu_inc * l):
            x = self.uzawa(lev, x, b)
        return x

    def solve(self, b, rtol=1e-8, max_cycles=100, x0=None):
        top = self.levels[0].prob
        x = np.zeros_like(b) if x0 is None else x0.copy()
        nb = np.linalg.norm(b)
        hist = [np.linalg.norm(b - top.apply(x)) / nb]
        for _ in range(max_cycles):
            x = self.vcycle(b, x)
            hist.append(np.linalg.norm(b - top.apply(x)) / nb)
            if hist[-1] <= rtol:
                break
        return top.gauge(x), hist

    def solve_krylov(self, b, rtol=1e-12, restart=30, maxiter=400):
        """GMRES(restart) (scipy, a library primitive) on the free-DoF system K_FF x = b_F,
        preconditioned by one V_var cycle from a zero guess: the outer iteration used
        when the plain V-cycle iteration does not converge (unresolved high-contrast
        inclusions).  Returns the gauged solution and the true relative
        residual."""
        import scipy.sparse.linalg as spla
        top = self.levels[0].prob
        free = np.flatnonzero(top.free)
        n4 = 4 * top.V
        if hasattr(top, "K"):
            Kf = top.K_free()
            matvec = Kf.__matmul__
        else:
            def matvec(v):
                x = np.zeros(n4)
                x[free] = v
                return top.apply(x)[free]

        def prec(r):
            full = np.zeros(n4)
            full[free] = r
            return self.vcycle(full, np.zeros(n4))[free]

        N = len(free)
        Aop = spla.LinearOperator((N, N), matvec=matvec)
        M = spla.LinearOperator((N, N), matvec=prec)
        xf, info = spla.gmres(Aop, b[free], M=M, rtol=rtol, atol=0.0, restart=restart, maxiter=maxiter)
        x = np.zeros(n4)
        x[free] = xf
        rel = np.linalg.norm(b - top.apply(x)) / np.linalg.norm(b)
        return top.gauge(x), rel
