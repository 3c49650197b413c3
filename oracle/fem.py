"""ORACLE (test infrastructure only) — element matrices and global assembly.

Plain definition of the discrete operators of PAPER.md, P1-P1 on the Kuhn
tetrahedral grid, by exact element-by-element integration (integrands are
constant or linear for P1) and textbook global assembly.  No stencils, no
blocking, no reordering.

Forms (velocity block A), test index (i,a) = row, trial index (j,b) = column:
  grad : (mu grad u, grad v)                 P:159 (volume term of a_int)
  sym  : (2 mu sym grad u, sym grad v)       P:151-153 (eq. standard)
  mod  : a_sym - (mu div u, div v)           P:199-203 (eq. newbil), "a_tr"
  dev  : (2 mu dev sym grad u, dev sym grad v)   P:205-207 (for checks only)
Divergence  b(v,q) = -(div v, q)
Stabilisation c(p,q) = sum_T (delta h^2 / mu_T) (grad p, grad q)_T
            (Brezzi-Pitkaranta type; constant and mu-weighting are the
             DESIGN.md reading R1 — the paper does not print the P1-P1 form)
            On coarse multigrid levels the viscosity of A and the 1/mu weight of C
            (and of the gauge) are separate per-element arrays (reading R15).
Saddle system  [[A, B^T], [B, -C]] (u, p) = (f_h, 0)   P:1222-1235.
Boundary: velocity DoFs on Dirichlet faces and the face-normal component on
free-slip faces (u.n = 0; the tangential traction condition is natural)
are eliminated; traction faces are natural.

Vectors are field-major: [u1 (V), u2 (V), u3 (V), p (V)], vertex
v = i + (n+1)(j + (n+1)k) (synth module convention).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from synth import PERMS, DIRICHLET, TRACTION, dirichlet_vertex_mask, eliminated_mask

FORMS = ("mod", "sym", "grad")


# ---------------------------------------------------------------------------
# element level
# ---------------------------------------------------------------------------
def kuhn_vertices(t: int) -> np.ndarray:
    """Vertices (units of h) of Kuhn tet t in the unit cube:
    a0 = 0, a1 = a0 + e_s1, a2 = a1 + e_s2, a3 = (1,1,1)."""
    s = PERMS[t]
    a = np.zeros((4, 3))
    a[1] = a[0]
    a[1, s[0]] += 1
    a[2] = a[1]
    a[2, s[1]] += 1
    a[3] = 1.0
    return a


def barycentric_gradients(verts: np.ndarray):
    """|T| and grad(lambda_i) (4x3) of the P1 hat functions on a tetrahedron.

    Plain definition: lambda_i(x) = c0 + c.x with lambda_i(a_j) = delta_ij, i.e.
    the columns of inv([[1, a_j^T]]_j)."""
    X = np.hstack([np.ones((4, 1)), verts])
    Cinv = np.linalg.inv(X)
    grads = Cinv[1:, :].T.copy()          # row i = grad lambda_i
    vol = abs(np.linalg.det(X)) / 6.0
    return vol, grads


def element_matrices(t: int, h: float, form: str):
    """Unit-coefficient element matrices of Kuhn tet t at mesh size h.

    Returns dict with
      A : 12x12, velocity block for mu = 1, local index a*4 + i
      B : 4x12,  B[i, b*4+j] = -(div (phi_j e_b), phi_i)_T = -|T|/4 dphi_j/dx_b
      C : 4x4,   (grad phi_i, grad phi_j)_T * h^2   (times delta/mu_T when assembled)
      M : 4x4,   consistent mass (phi_i, phi_j)_T
      D : 12x12, (div u, div v)_T for mu = 1
      vol, grads
    """
    vol, g = barycentric_gradients(kuhn_vertices(t) * h)
    A = np.zeros((12, 12))
    D = np.zeros((12, 12))
    S = np.zeros((12, 12))   # (grad u^T : grad v)
    G = np.zeros((12, 12))   # (grad u : grad v)
    for a in range(3):
        for i in range(4):
            r = a * 4 + i
            for b in range(3):
                for j in range(4):
                    c = b * 4 + j
                    # u = phi_j e_b (trial), v = phi_i e_a (test)
                    # (grad u)_{cd} = delta_cb dphi_j/dx_d ; (grad v)_{cd} = delta_ca dphi_i/dx_d
                    G[r, c] = vol * (g[i] @ g[j]) * (a == b)
                    S[r, c] = vol * g[j, a] * g[i, b]          # grad u^T : grad v
                    D[r, c] = vol * g[j, b] * g[i, a]          # div u * div v
    if form == "grad":
        A = G
    elif form == "sym":
        A = G + S                                              # 2 sym:sym = G + S
    elif form == "mod":
        A = G + S - D
    elif form == "dev":
        A = G + S - (2.0 / 3.0) * D                            # 2 dev sym : dev sym
    else:
        raise ValueError(form)
    B = np.zeros((4, 12))
    for i in range(4):
        for b in range(3):
            for j in range(4):
                B[i, b * 4 + j] = -(vol / 4.0) * g[j, b]
    C = vol * (g @ g.T) * h * h
    M = vol / 20.0 * (np.ones((4, 4)) + np.eye(4))
    return dict(A=A, B=B, C=C, M=M, D=D, vol=vol, grads=g)


# ---------------------------------------------------------------------------
# grid level
# ---------------------------------------------------------------------------
def _element_vertex_ids(n: int, t: int) -> np.ndarray:
    """Global vertex ids (n^3, 4) of the local vertices of tet t of every cube,
    cubes ordered [k][j][i]."""
    idx = np.arange(n)
    k, j, i = np.meshgrid(idx, idx, idx, indexing="ij")
    off = kuhn_vertices(t).astype(np.int64)
    N1 = n + 1
    out = np.empty((n ** 3, 4), dtype=np.int64)
    for m in range(4):
        out[:, m] = ((i + off[m, 0]) + N1 * ((j + off[m, 1]) + N1 * (k + off[m, 2]))).reshape(-1)
    return out


class Problem:
    """One grid level: n, element viscosities, faces, form, delta."""

    def __init__(self, n: int, elem_mu: np.ndarray, faces, form: str = "mod",
                 delta: float = 1.0 / 12.0, elem_imu_c: np.ndarray | None = None):
        """elem_mu: mu_T of the viscous block A per element [k][j][i][t];
        elem_imu_c: the 1/mu_T weight of C and of the gauge (default 1/elem_mu;
        coarse levels pass their own, reading R15)."""
        self.n = n
        self.h = 1.0 / n
        self.V = (n + 1) ** 3
        self.elem_mu = np.asarray(elem_mu, dtype=np.float64).reshape(n, n, n, 6)
        self.elem_imu_c = (1.0 / self.elem_mu if elem_imu_c is None else
                           np.asarray(elem_imu_c, dtype=np.float64).reshape(n, n, n, 6))
        self.faces = tuple(faces)
        self.form = form
        self.delta = delta
        self.dir_v = dirichlet_vertex_mask(n, self.faces)
        # eliminated velocity DoFs: Dirichlet faces and the normal component on
        # free-slip faces (u.n = 0); their rows and columns are dropped
        self.elim = eliminated_mask(n, self.faces)
        self.free = np.concatenate([~self.elim.reshape(-1), np.ones(self.V, dtype=bool)])
        self.has_traction = any(f == TRACTION for f in self.faces)
        self._assemble()

    def _assemble(self):
        n, V = self.n, self.V
        rowsA, colsA, valsA = [], [], []
        rowsB, colsB, valsB = [], [], []
        rowsC, colsC, valsC = [], [], []
        rowsM, colsM, valsM = [], [], []
        w = np.zeros(V)
        for t in range(6):
            em = element_matrices(t, self.h, self.form)
            vid = _element_vertex_ids(n, t)                    # (E,4)
            mu = self.elem_mu[..., t].reshape(-1)              # (E,)
            imu = self.elem_imu_c[..., t].reshape(-1)          # (E,)
            gidx = np.concatenate([vid + a * V for a in range(3)], axis=1)   # (E,12)
            rowsA.append(np.repeat(gidx, 12, axis=1).reshape(-1))
            colsA.append(np.tile(gidx, (1, 12)).reshape(-1))
            valsA.append((mu[:, None] * em["A"].reshape(1, -1)).reshape(-1))
            rowsB.append(np.repeat(vid, 12, axis=1).reshape(-1))
            colsB.append(np.tile(gidx, (1, 4)).reshape(-1))
            valsB.append(np.broadcast_to(em["B"].reshape(1, -1), (len(mu), 48)).reshape(-1))
            rowsC.append(np.repeat(vid, 4, axis=1).reshape(-1))
            colsC.append(np.tile(vid, (1, 4)).reshape(-1))
            valsC.append(((self.delta * imu)[:, None] * em["C"].reshape(1, -1)).reshape(-1))
            rowsM.append(rowsC[-1])
            colsM.append(colsC[-1])
            valsM.append(np.broadcast_to(em["M"].reshape(1, -1), (len(mu), 16)).reshape(-1))
            np.add.at(w, vid.reshape(-1), np.repeat(em["vol"] * imu / 4.0, 4))
        cat = np.concatenate
        self.A = sp.csr_matrix((cat(valsA), (cat(rowsA), cat(colsA))), shape=(3 * V, 3 * V))
        self.B = sp.csr_matrix((cat(valsB), (cat(rowsB), cat(colsB))), shape=(V, 3 * V))
        self.C = sp.csr_matrix((cat(valsC), (cat(rowsC), cat(colsC))), shape=(V, V))
        self.M = sp.csr_matrix((cat(valsM), (cat(rowsM), cat(colsM))), shape=(V, V))
        for m in (self.A, self.B, self.C, self.M):
            m.sum_duplicates()
        self.K = sp.bmat([[self.A, self.B.T], [self.B, -self.C]], format="csr")
        self.gauge_w = w      # w_j = int phi_j / mu  (discrete int mu^-1 p = 0)

    # -- operator on free DoFs -------------------------------------------
    def apply(self, x: np.ndarray) -> np.ndarray:
        """y = K_FF x_F, Dirichlet inputs ignored, Dirichlet outputs 0 (field-major 4V)."""
        xf = np.where(self.free, x.reshape(-1), 0.0)
        return np.where(self.free, self.K @ xf, 0.0)

    def K_free(self) -> sp.csr_matrix:
        idx = np.flatnonzero(self.free)
        return self.K[idx][:, idx].tocsr()

    # -- load vectors (reading R10) ------------------------------
    def load_nodal(self, f: np.ndarray) -> np.ndarray:
        """b_u = (M (x) I3) f, b_p = 0, zero at Dirichlet rows."""
        f = f.reshape(3, self.V)
        b = np.concatenate([self.M @ f[a] for a in range(3)] + [np.zeros(self.V)])
        return np.where(self.free, b, 0.0)

    def load_element(self, f_elem: np.ndarray) -> np.ndarray:
        """Element-constant f: b_{i,a} = sum_{T ni i} f_{T,a} |T|/4; f_elem (E6, 3)."""
        n, V = self.n, self.V
        f_elem = np.asarray(f_elem).reshape(n, n, n, 6, 3)
        b = np.zeros((3, V))
        vol = self.h ** 3 / 6.0
        for t in range(6):
            vid = _element_vertex_ids(n, t)
            ft = f_elem[..., t, :].reshape(-1, 3)
            for a in range(3):
                np.add.at(b[a], vid.reshape(-1), np.repeat(ft[:, a] * vol / 4.0, 4))
        out = np.concatenate([b.reshape(-1), np.zeros(V)])
        return np.where(self.free, out, 0.0)

    # -- gauge -------------------------------------------------------------
    def gauge(self, x: np.ndarray) -> np.ndarray:
        """Subtract the mu^-1-weighted mean pressure (Q of P:136); no-op with traction."""
        x = x.copy().reshape(-1)
        if self.has_traction:
            return x
        p = x[3 * self.V:]
        x[3 * self.V:] = p - (self.gauge_w @ p) / self.gauge_w.sum()
        return x

    # -- direct solve -------------------------------------------------------
    def solve_direct(self, b: np.ndarray, x_dir: np.ndarray | None = None) -> np.ndarray:
        """Unique discrete solution of K_FF x_F = b_F (- K_FD x_D), gauged.

        Without a traction face K_FF has the constant pressure as its null vector
         and b_p = 0 is consistent with it: the last pressure unknown is pinned
        to 0 (its row and column removed -- the removed equation holds by
        consistency), the reduced nonsingular system is solved directly (sparse LU),
        and the result is gauged to int mu^-1 p = 0 (reading R9)."""
        import scipy.sparse.linalg as spla
        free = np.flatnonzero(self.free)
        rhs = b.reshape(-1)[free].copy()
        if x_dir is not None:
            xd = np.where(self.free, 0.0, x_dir.reshape(-1))
            rhs -= (self.K @ xd)[free]
        Kff = self.K[free][:, free].tocsc()
        keep = np.arange(len(free))
        if not self.has_traction:
            keep = keep[:-1]                      # free[-1] is the last pressure DoF
            Kff = Kff[keep][:, keep]
        sol = np.zeros(len(free))
        sol[keep] = spla.spsolve(Kff.tocsc(), rhs[keep])
        x = np.zeros(4 * self.V) if x_dir is None else np.where(self.free, 0.0, x_dir.reshape(-1))
        x[free] = sol
        return self.gauge(x)


def load_nodal_elementwise(n: int, faces, f: np.ndarray) -> np.ndarray:
    """b_u = (M (x) I3) f by the element loop (consistent P1 mass |T|/20 (1 + d_ij) per
    tet, no assembled matrix: for the matrix-free oracle levels); b_p = 0; zero at
    Dirichlet rows.  Equals Problem.load_nodal (pinned by the mass-stencil test)."""
    V = (n + 1) ** 3
    f = np.asarray(f, dtype=np.float64).reshape(3, V)
    vol = (1.0 / n) ** 3 / 6.0
    b = np.zeros((3, V))
    for t in range(6):
        vid = _element_vertex_ids(n, t)                    # (E, 4)
        for a in range(3):
            fl = f[a][vid]                                 # (E, 4)
            loc = (vol / 20.0) * (fl.sum(axis=1, keepdims=True) + fl)
            b[a] += np.bincount(vid.reshape(-1), weights=loc.reshape(-1), minlength=V)
    b[eliminated_mask(n, faces)] = 0.0
    return np.concatenate([b.reshape(-1), np.zeros(V)])


def problem_from_classes(n, mu_cls, class_mu, faces, form="mod", delta=1.0 / 12.0):
    elem_mu = np.asarray(class_mu, dtype=np.float64)[np.asarray(mu_cls)]
    return Problem(n, elem_mu, faces, form, delta)


def element_force(n, f_cls, force_table):
    return np.asarray(force_table, dtype=np.float64)[np.asarray(f_cls)]
