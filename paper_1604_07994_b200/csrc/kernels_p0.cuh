// The stabilised P1-P0 operator (§3.3-3.4): P1 velocity
// as everywhere else, one pressure per tetrahedron,
//   b(v, q) = -(div v, q)
//   c(p, q) = gamma sum_i 1/(2 mu_i) sum_{F interior facet of Omega_i}
//             |T1||T2|/(|T1|+|T2|) [p][q]                             (eq. stabc)
// (no jump penalised across Gamma_12 or on the boundary), K0 = [[A, B0^T], [B0, -C0]]
// (P:431-438).  The A block is the library's (stk_apply, blocks = A); two kernels add
// the P0 couplings:
//  * k_p0_bt: per vertex, (B0^T p)_{v,a} = -sum_{T ni v} |T| (grad lambda_m)_a p_T over
//    the 24 incident Kuhn tets (eliminated velocity components 0);
//  * k_p0_rows: per tet, (B0 u)_T - (C0 p)_T = -|T| div u_T - sum_F w_F (p_T - p_T'),
//    facet neighbours from the compile-time Kuhn face table below, w_F = gamma / (2 mu)
//    * |T|/2 (uniform Kuhn grid: all tets have |T| = h^3 / 6) when both tets carry the
//    same viscosity.
// Pressure layout: element order of the classes (e = 6 (i + n (j + n k)) + t), fp64.
#pragma once
#include "stk_common.cuh"

namespace stk {

// face neighbour of Kuhn tet t across the face opposite its local vertex m: cube
// offset (dx, dy, dz) and tet t' (every face of the Kuhn split has exactly one
// neighbour in the 3x3x3 cube neighbourhood; on the cube boundary it lies outside)
struct FnbTab {
  int8_t dx[6][4], dy[6][4], dz[6][4], tn[6][4];
};
__host__ __device__ constexpr bool p0_has_vertex(int ox, int oy, int oz, int t, int px, int py, int pz) {
  bool r = false;
  for (int q = 0; q < 4; ++q) {
    const int c = ktet_corner(t, q);
    if (ox + (c & 1) == px && oy + ((c >> 1) & 1) == py && oz + (c >> 2) == pz) r = true;
  }
  return r;
}
__host__ __device__ constexpr FnbTab make_fnb() {
  FnbTab T{};
  for (int t = 0; t < 6; ++t)
    for (int m = 0; m < 4; ++m) {
      int P[3][3] = {};
      int w = 0;
      for (int q = 0; q < 4; ++q) {
        if (q == m) continue;
        const int c = ktet_corner(t, q);
        P[w][0] = c & 1;
        P[w][1] = (c >> 1) & 1;
        P[w][2] = c >> 2;
        ++w;
      }
      T.tn[t][m] = -1;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx)
            for (int u = 0; u < 6; ++u) {
              if (dx == 0 && dy == 0 && dz == 0 && u == t) continue;
              bool all = true;
              for (int k = 0; k < 3; ++k)
                all = all && p0_has_vertex(dx, dy, dz, u, P[k][0], P[k][1], P[k][2]);
              if (all) {
                T.dx[t][m] = (int8_t)dx;
                T.dy[t][m] = (int8_t)dy;
                T.dz[t][m] = (int8_t)dz;
                T.tn[t][m] = (int8_t)u;
              }
            }
    }
  return T;
}
constexpr FnbTab kFnb = make_fnb();
constexpr bool fnb_ok() {
  for (int t = 0; t < 6; ++t)
    for (int m = 0; m < 4; ++m) {
      if (kFnb.tn[t][m] < 0) return false;
      // symmetric: the neighbour's neighbour across the shared face is t
      const int u = kFnb.tn[t][m];
      bool back = false;
      for (int m2 = 0; m2 < 4; ++m2)
        if (kFnb.tn[u][m2] == t && kFnb.dx[u][m2] == -kFnb.dx[t][m] && kFnb.dy[u][m2] == -kFnb.dy[t][m] &&
            kFnb.dz[u][m2] == -kFnb.dz[t][m])
          back = true;
      if (!back) return false;
    }
  return true;
}
static_assert(fnb_ok(), "Kuhn face-neighbour table");
__constant__ FnbTab c_fnb = make_fnb();

// grad lambda_m of Kuhn tet t (units 1/h): -e_s1 (m=0), e_s1 - e_s2, e_s2 - e_s3, e_s3 (m=3)
__device__ __forceinline__ void p0_grad(int t, int m, double hinv, double g[3]) {
  const int s1 = kperm(t, 0), s2 = kperm(t, 1), s3 = kperm(t, 2);
  g[0] = g[1] = g[2] = 0.0;
  if (m == 0) g[s1] = -hinv;
  else if (m == 1) { g[s1] = hinv; g[s2] = -hinv; }
  else if (m == 2) { g[s2] = hinv; g[s3] = -hinv; }
  else g[s3] = hinv;
}

// y_u += B0^T p at every owned vertex (velocity fields of the padded level vector)
__global__ void k_p0_bt(DGrid g, const double* __restrict__ p0, double* __restrict__ y) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const double hinv = 1.0 / g.h, vol = g.h * g.h * g.h / 6.0;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int own = 0; own < 8; ++own) {
    const int ci = i - (own & 1), cj = j - ((own >> 1) & 1), ck = k - (own >> 2);
    if (ci < 0 || cj < 0 || ck < 0 || ci >= g.n || cj >= g.n || ck >= g.n) continue;
    for (int t = 0; t < 6; ++t) {
      const int m = kcorner(own, t);
      if (m < 0) continue;
      double gm[3];
      p0_grad(t, m, hinv, gm);
      const double pt = p0[((((int64_t)ck * g.n) + cj) * g.n + ci) * 6 + t];
#pragma unroll
      for (int a = 0; a < 3; ++a) acc[a] -= vol * gm[a] * pt;
    }
  }
  const unsigned em = elim(g, i, j, k);
  const int64_t o = vidx(g, i, j, k);
#pragma unroll
  for (int a = 0; a < 3; ++a) y[a * g.fs + o] = ((em >> a) & 1u) ? 0.0 : y[a * g.fs + o] + acc[a];
}

// y0_T = (B0 u)_T - (C0 p)_T for every tet (u: velocity fields of the padded level vector,
// eliminated entries 0)
__global__ void k_p0_rows(DGrid g, const double* __restrict__ u, const double* __restrict__ p0,
                          double* __restrict__ y0, double gamma) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = g.n;
  if (e >= (int64_t)6 * n * n * n) return;
  const int t = (int)(e % 6);
  int64_t r = e / 6;
  const int ci = (int)(r % n);
  r /= n;
  const int cj = (int)(r % n), ck = (int)(r / n);
  const double hinv = 1.0 / g.h, vol = g.h * g.h * g.h / 6.0;
  double div = 0.0;
  for (int m = 0; m < 4; ++m) {
    const int c = ktet_corner(t, m);
    const int vi = ci + (c & 1), vj = cj + ((c >> 1) & 1), vk = ck + (c >> 2);
    const int64_t o = vidx(g, vi, vj, vk);
    double gm[3];
    p0_grad(t, m, hinv, gm);
    div += gm[0] * u[o] + gm[1] * u[g.fs + o] + gm[2] * u[2 * g.fs + o];
  }
  const int cl = elem_class(g, ci, cj, ck, t);
  const double mu = mu_of(g, cl);
  const double w = gamma / (2.0 * mu) * (0.5 * vol);  // |T1||T2|/(|T1|+|T2|) = |T|/2
  const double pt = p0[e];
  double cp = 0.0;
  for (int m = 0; m < 4; ++m) {
    const int ni = ci + c_fnb.dx[t][m], nj = cj + c_fnb.dy[t][m], nk = ck + c_fnb.dz[t][m];
    if (ni < 0 || nj < 0 || nk < 0 || ni >= n || nj >= n || nk >= n) continue;  // boundary facet
    const int tn = c_fnb.tn[t][m];
    if (mu_of(g, elem_class(g, ni, nj, nk, tn)) != mu) continue;  // facet on Gamma_12: no penalty
    cp += w * (pt - p0[((((int64_t)nk * n) + nj) * n + ni) * 6 + tn]);
  }
  y0[e] = -vol * div - cp;
}

// auxiliary-space maps between the P0 and the P1 pressure (stk_p0_solve's
// preconditioner): a P0 residual (per-tet integrals) is shared equally by the tet's 4
// vertices -- the transpose of the tet average -- and a P1 correction is averaged over
// each tet's 4 vertices
__global__ void k_p0_to_p1(DGrid g, const double* __restrict__ r0, double* __restrict__ bp) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  double acc = 0.0;
  for (int own = 0; own < 8; ++own) {
    const int ci = i - (own & 1), cj = j - ((own >> 1) & 1), ck = k - (own >> 2);
    if (ci < 0 || cj < 0 || ck < 0 || ci >= g.n || cj >= g.n || ck >= g.n) continue;
    for (int t = 0; t < 6; ++t)
      if (kcorner(own, t) >= 0) acc += 0.25 * r0[((((int64_t)ck * g.n) + cj) * g.n + ci) * 6 + t];
  }
  bp[vidx(g, i, j, k)] = acc;
}
// (r0 != nullptr: plus the element-local Schur-complement term -wp (mu_T / |T|) r0, the
// 1/mu-weighted P0 mass inverse -- it reaches the per-tet pressure modes the P1 auxiliary
// space cannot represent; without it the preconditioner is singular on them and GMRES
// stagnates near 1e-3)
__global__ void k_p1_to_p0(DGrid g, const double* __restrict__ zp, double* __restrict__ z0,
                           const double* __restrict__ r0 = nullptr, double wp = 0.0) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = g.n;
  if (e >= (int64_t)6 * n * n * n) return;
  const int t = (int)(e % 6);
  int64_t r = e / 6;
  const int ci = (int)(r % n);
  r /= n;
  const int cj = (int)(r % n), ck = (int)(r / n);
  double s = 0.0;
  for (int q = 0; q < 4; ++q) {
    const int c = ktet_corner(t, q);
    s += zp[vidx(g, ci + (c & 1), cj + ((c >> 1) & 1), ck + (c >> 2))];
  }
  double z = 0.25 * s;
  if (r0) z -= wp * mu_of(g, elem_class(g, ci, cj, ck, t)) * (6.0 / (g.h * g.h * g.h)) * r0[e];
  z0[e] = z;
}

// local flux post-process: flux[4 e + m] = int_F j_{F;T} over the facet of
// tet e opposite its local vertex m: int_F u_h . n_T = -|T| grad lambda_m . sum_{q != m} u_q
// (|F| = 3 |T| |grad lambda_m|, n_T = -grad lambda_m / |grad lambda_m|, the facet mean of
// a P1 field is the mean of its 3 vertices), plus w_F (p_T - p_T') on facets interior to
// one subdomain.  sum_m flux[4 e + m] = |T| div u_T + sum_F w_F (p_T - p_T') = -(B0 u -
// C0 p)_T: zero at a discrete solution with zero mass rhs (element-wise conservation).
__global__ void k_p0_fluxes(DGrid g, const double* __restrict__ u, const double* __restrict__ p0,
                            double* __restrict__ flux, double gamma) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = g.n;
  if (e >= (int64_t)6 * n * n * n) return;
  const int t = (int)(e % 6);
  int64_t r = e / 6;
  const int ci = (int)(r % n);
  r /= n;
  const int cj = (int)(r % n), ck = (int)(r / n);
  const double hinv = 1.0 / g.h, vol = g.h * g.h * g.h / 6.0;
  double uq[4][3];
  for (int q = 0; q < 4; ++q) {
    const int c = ktet_corner(t, q);
    const int64_t o = vidx(g, ci + (c & 1), cj + ((c >> 1) & 1), ck + (c >> 2));
    for (int a = 0; a < 3; ++a) uq[q][a] = u[a * g.fs + o];
  }
  const double mu = mu_of(g, elem_class(g, ci, cj, ck, t));
  const double w = gamma / (2.0 * mu) * (0.5 * vol);
  const double pt = p0[e];
  for (int m = 0; m < 4; ++m) {
    double gm[3];
    p0_grad(t, m, hinv, gm);
    double s = 0.0;
    for (int q = 0; q < 4; ++q)
      if (q != m) s += gm[0] * uq[q][0] + gm[1] * uq[q][1] + gm[2] * uq[q][2];
    double f = -vol * s;
    const int ni = ci + c_fnb.dx[t][m], nj = cj + c_fnb.dy[t][m], nk = ck + c_fnb.dz[t][m];
    if (ni >= 0 && nj >= 0 && nk >= 0 && ni < n && nj < n && nk < n) {
      const int tn = c_fnb.tn[t][m];
      if (mu_of(g, elem_class(g, ni, nj, nk, tn)) == mu) f += w * (pt - p0[((((int64_t)nk * n) + nj) * n + ni) * 6 + tn]);
    }
    flux[4 * e + m] = f;
  }
}

}  // namespace stk
