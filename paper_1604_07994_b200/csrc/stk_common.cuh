// Common device definitions of the B200 Stokes library (sm_100a, fp64).
//
// Grid: unit cube, n^3 cubes, each split into the 6 Kuhn tetrahedra
//   t <-> sigma in {(x,y,z),(x,z,y),(y,x,z),(y,z,x),(z,x,y),(z,y,x)}
//   a0 = c, a1 = a0 + h e_s1, a2 = a1 + h e_s2, a3 = c + h(1,1,1)
// which is the six-tetrahedra split of P:720; uniform (Bey) refinement of this
// mesh is the same Kuhn grid at h/2, so every level is structured.
//
// Layout of a level vector (z-slab of this rank): 4 fields (u1,u2,u3,p),
//   f*fs + (k - z0 + 1)*py + (j + 1)*px + (i + 1)
// planes z0-1 and z0+nzl are halos; column i = -1 and row j = -1 are a zero
// ghost frame so that every TMA box starts at non-negative coordinates.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace stk {

enum { FORM_MOD = 0, FORM_SYM = 1, FORM_GRAD = 2 };
enum { BLK_A = 1, BLK_BT = 2, BLK_B = 4, BLK_C = 8, BLK_ALL = 15 };
constexpr uint8_t CODE_IRREGULAR = 0xFF;
// element class of a coarse tet whose Bey children do not share one class
// (reading R15): its coefficients are the per-tet means in DGrid::emu
constexpr uint8_t CLS_MIXED = 0xFE;

// Kuhn permutations
__constant__ int8_t c_perm[6][3];
// local index (0..3) of cube corner `corner` (bit0 x, bit1 y, bit2 z) in tet t, or -1
__constant__ int8_t c_corner_m[8][6];
// Bey children of a coarse tet T: fine cube offset (bits x|y<<1|z<<2) and fine type
__constant__ int8_t c_child_off[6][8];
__constant__ int8_t c_child_t[6][8];

// compile-time Kuhn tables (the __constant__ copies above serve the setup kernels)
__host__ __device__ constexpr int kperm(int t, int q) {
  return t == 0 ? (q == 0 ? 0 : q == 1 ? 1 : 2)
       : t == 1 ? (q == 0 ? 0 : q == 1 ? 2 : 1)
       : t == 2 ? (q == 0 ? 1 : q == 1 ? 0 : 2)
       : t == 3 ? (q == 0 ? 1 : q == 1 ? 2 : 0)
       : t == 4 ? (q == 0 ? 2 : q == 1 ? 0 : 1)
                : (q == 0 ? 2 : q == 1 ? 1 : 0);
}
// local index of cube corner c (bit0 x, bit1 y, bit2 z) in Kuhn tet t, or -1
__host__ __device__ constexpr int kcorner(int c, int t) {
  return c == 0 ? 0
       : c == 7 ? 3
       : c == (1 << kperm(t, 0)) ? 1
       : c == ((1 << kperm(t, 0)) | (1 << kperm(t, 1))) ? 2
                                                        : -1;
}

struct DGrid {
  int n;            // intervals of this level
  int z0, nzl;      // owned vertex planes [z0, z0+nzl)
  int cz0;          // first stored cube layer
  int64_t px, py, fs;
  double h;
  double delta;     // stabilisation constant
  double idh3;      // 1 / (delta h^3)
  unsigned dirmask; // bit f set: face f is homogeneous Dirichlet
  unsigned slipmask; // bit f set: face f is free-slip (u.n = 0, tangential traction 0)
  const uint8_t* cls;   // element classes [cz - cz0][cj][ci][t]
  const uint8_t* code;  // per-vertex code (plane layout of one field)
  const double* mu;     // per-class viscosity mu_k [0..255], 1/mu_k at mu + 256 (device)
  // coarse levels: per-tet (mu_A, 1/mu_C) means over the Bey children (reading R15), same
  // layout as cls; read for CLS_MIXED tets only (a pure tet's pair is its class's)
  const double2* emu;
};

__device__ __forceinline__ double mu_of(const DGrid& g, int cl) { return __ldg(g.mu + cl); }
// the same per-class table as a kernel parameter (constant bank): the latency-bound
// coarse-level row kernels read mu without a dependent L2 round trip
struct MuTab {
  double mu[256], imu[256];
};
__device__ __forceinline__ double imu_of(const DGrid& g, int cl) { return __ldg(g.mu + 256 + cl); }

__device__ __forceinline__ int64_t vidx(const DGrid& g, int i, int j, int k) {
  return (int64_t)(k - g.z0 + 1) * g.py + (int64_t)(j + 1) * g.px + (i + 1);
}
inline int64_t vidx_host(const DGrid& g, int i, int j, int k) {
  return (int64_t)(k - g.z0 + 1) * g.py + (int64_t)(j + 1) * g.px + (i + 1);
}

__device__ __forceinline__ bool is_dirichlet(const DGrid& g, int i, int j, int k) {
  const unsigned m = g.dirmask;
  return ((m & 1u) && i == 0) || ((m & 2u) && i == g.n) || ((m & 4u) && j == 0) ||
         ((m & 8u) && j == g.n) || ((m & 16u) && k == 0) || ((m & 32u) && k == g.n);
}

// eliminated velocity components of vertex (i,j,k): bit a = component a is fixed to 0
// (all three on a Dirichlet face; the face-normal component on a free-slip face,
// u.n = 0; Dirichlet wins on shared edges and corners)
__host__ __device__ __forceinline__ unsigned elim_mask(unsigned dm, unsigned sm, int n, int i, int j, int k) {
  const unsigned onf = (i == 0 ? 1u : 0u) | (i == n ? 2u : 0u) | (j == 0 ? 4u : 0u) | (j == n ? 8u : 0u) |
                       (k == 0 ? 16u : 0u) | (k == n ? 32u : 0u);
  if (onf & dm) return 7u;
  const unsigned s = onf & sm;
  return ((s & 3u) ? 1u : 0u) | ((s & 12u) ? 2u : 0u) | ((s & 48u) ? 4u : 0u);
}
__device__ __forceinline__ unsigned elim(const DGrid& g, int i, int j, int k) {
  return elim_mask(g.dirmask, g.slipmask, g.n, i, j, k);
}

__device__ __forceinline__ int64_t elem_index(const DGrid& g, int ci, int cj, int ck, int t) {
  return ((((int64_t)(ck - g.cz0)) * g.n + cj) * g.n + ci) * 6 + t;
}
__device__ __forceinline__ uint8_t elem_class(const DGrid& g, int ci, int cj, int ck, int t) {
  return g.cls[elem_index(g, ci, cj, ck, t)];
}
// (mu_A, 1/mu_C) of tet (ci,cj,ck,t) with class cl: the class table, or the per-tet
// coarse-level means of a MIXED tet (reading R15)
__device__ __forceinline__ void tet_coef(const DGrid& g, int ci, int cj, int ck, int t, int cl, double& mu,
                                         double& imu) {
  if (cl == CLS_MIXED) {
    const double2 e = __ldg(g.emu + elem_index(g, ci, cj, ck, t));
    mu = e.x;
    imu = e.y;
  } else {
    mu = mu_of(g, cl);
    imu = imu_of(g, cl);
  }
}

// Generic row of K = [[A, B^T], [B, -C]] at owned vertex (i,j,k), by the
// element loop over its 24 incident tetrahedra (exact P1 integration):
//   (A u)_{i,a} = sum_T mu_T |T| [(G + G^T - tr(G) I) g_m]_a      (mod)
//                 sum_T mu_T |T| [(G + G^T) g_m]_a               (sym)
//                 sum_T mu_T |T| [G g_m]_a                       (grad)
//   (B^T p)_{i,a} = -sum_T |T|/4 g_m[a] sum_{q in T} p_q
//   (B u)_i       = -sum_T |T|/4 tr(G)
//   (C p)_i       =  sum_T delta h^2/mu_T |T| g_m . grad p        (DESIGN R1)
// G = grad u on T from the Kuhn path differences, g_m = grad lambda_m.
// Also returns the diagonals of A (per component) and C (for Gauss-Seidel).
template <int FORM, class F>
__device__ __forceinline__ void row_generic(const DGrid& g, int i, int j, int k, const F& fx,
                                            unsigned blocks, double y[4], double dA[3],
                                            double& dC) {
  const double h = g.h, hinv = 1.0 / h;
  const double vol = h * h * h / 6.0, vq = 0.25 * vol;
  const double cstab = g.delta * h * h * vol;
  y[0] = y[1] = y[2] = y[3] = 0.0;
  dA[0] = dA[1] = dA[2] = 0.0;
  dC = 0.0;
#pragma unroll
  for (int dz = -1; dz <= 0; ++dz) {
    const int ck = k + dz;
    if (ck < 0 || ck >= g.n) continue;
#pragma unroll
    for (int dy = -1; dy <= 0; ++dy) {
      const int cj = j + dy;
      if (cj < 0 || cj >= g.n) continue;
#pragma unroll
      for (int dx = -1; dx <= 0; ++dx) {
        const int ci = i + dx;
        if (ci < 0 || ci >= g.n) continue;
        const int corner = (-dx) | ((-dy) << 1) | ((-dz) << 2);
#pragma unroll
        for (int t = 0; t < 6; ++t) {
          const int m = kcorner(corner, t);
          if (m < 0) continue;
          const int s1 = kperm(t, 0), s2 = kperm(t, 1), s3 = kperm(t, 2);
          int v[4][3];
          v[0][0] = ci; v[0][1] = cj; v[0][2] = ck;
          v[1][0] = ci; v[1][1] = cj; v[1][2] = ck; v[1][s1] += 1;
          v[2][0] = v[1][0]; v[2][1] = v[1][1]; v[2][2] = v[1][2]; v[2][s2] += 1;
          v[3][0] = ci + 1; v[3][1] = cj + 1; v[3][2] = ck + 1;
          double val[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int f = 0; f < 4; ++f) val[q][f] = fx(g, v[q][0], v[q][1], v[q][2], f);
          double G[3][3], gp[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            G[a][s1] = (val[1][a] - val[0][a]) * hinv;
            G[a][s2] = (val[2][a] - val[1][a]) * hinv;
            G[a][s3] = (val[3][a] - val[2][a]) * hinv;
          }
          gp[s1] = (val[1][3] - val[0][3]) * hinv;
          gp[s2] = (val[2][3] - val[1][3]) * hinv;
          gp[s3] = (val[3][3] - val[2][3]) * hinv;
          double gm[3] = {0.0, 0.0, 0.0};
          if (m == 0) {
            gm[s1] = -hinv;
          } else if (m == 1) {
            gm[s1] = hinv; gm[s2] = -hinv;
          } else if (m == 2) {
            gm[s2] = hinv; gm[s3] = -hinv;
          } else {
            gm[s3] = hinv;
          }
          const uint8_t cl = elem_class(g, ci, cj, ck, t);
          double mu, imu;
          tet_coef(g, ci, cj, ck, t, cl, mu, imu);
          const double gg = gm[0] * gm[0] + gm[1] * gm[1] + gm[2] * gm[2];
          const double tr = G[0][0] + G[1][1] + G[2][2];
          if (blocks & BLK_A) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              double s = G[a][0] * gm[0] + G[a][1] * gm[1] + G[a][2] * gm[2];
              if (FORM != FORM_GRAD) s += G[0][a] * gm[0] + G[1][a] * gm[1] + G[2][a] * gm[2];
              if (FORM == FORM_MOD) s -= tr * gm[a];
              y[a] += mu * vol * s;
            }
          }
          if (blocks & BLK_BT) {
            const double ps = val[0][3] + val[1][3] + val[2][3] + val[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a) y[a] -= vq * gm[a] * ps;
          }
          if (blocks & BLK_B) y[3] -= vq * tr;
          if (blocks & BLK_C) y[3] -= cstab * imu * (gm[0] * gp[0] + gm[1] * gp[1] + gm[2] * gp[2]);
#pragma unroll
          for (int a = 0; a < 3; ++a)
            dA[a] += mu * vol * (gg + (FORM == FORM_SYM ? gm[a] * gm[a] : 0.0));
          dC += cstab * imu * gg;
        }
      }
    }
  }
  {
    const unsigned em = elim(g, i, j, k);
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if ((em >> a) & 1u) y[a] = 0.0;
  }
}

// local cube corner (bit0 x, bit1 y, bit2 z) of vertex q = 0..3 of Kuhn tet t
__host__ __device__ constexpr int ktet_corner(int t, int q) {
  return q == 0 ? 0 : q == 1 ? (1 << kperm(t, 0)) : q == 2 ? ((1 << kperm(t, 0)) | (1 << kperm(t, 1))) : 7;
}
// is cube corner c a vertex of some tet of the cube that contains corner `own`?
__host__ __device__ constexpr bool kcube_needs(int own, int c) {
  bool r = false;
  for (int t = 0; t < 6; ++t)
    if (kcorner(own, t) >= 0 && kcorner(c, t) >= 0) r = true;
  return r;
}

// The same row as row_generic, for rows read from global memory (the list rows
// of the tiled kernels): the 15-point Kuhn neighbourhood (4 fields) and the
// classes of the 24 star tets are loaded up front (one round of memory
// latency, all loads independent), then the tets are integrated cube-major from
// registers.  U: velocity fields 0..2 (stride fs; 0 at Dirichlet vertices and
// outside the cube), Pf: pressure field.  PRED: pressure taken only at colour-0
// vertices ((i+j+k) even; the masked T of the pressure Gauss-Seidel, P:1243 /
// DESIGN R11) and no velocity.
template <int FORM, bool PRED>
__device__ __forceinline__ void row_list(const DGrid& g, int i, int j, int k, const double* __restrict__ U,
                                         const double* __restrict__ Pf, unsigned blocks, double y[4], double dA[3],
                                         double& dC) {
  const double h = g.h, hinv = 1.0 / h;
  const double vol = h * h * h / 6.0, vq = 0.25 * vol;
  const double cstab = g.delta * h * h * vol;
  const unsigned dm = g.dirmask;
  const int n = g.n;
  const int64_t o0 = vidx(g, i, j, k);
  // neighbourhood values nb[o][f], o = (dz+1)*9 + (dy+1)*3 + (dx+1), Kuhn offsets only
  double nb[27][4];
#pragma unroll
  for (int o = 0; o < 27; ++o) {
    const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
    if (!((dx >= 0 && dy >= 0 && dz >= 0) || (dx <= 0 && dy <= 0 && dz <= 0))) continue;
    const int xi = i + dx, yj = j + dy, zk = k + dz;
    const bool in = xi >= 0 && yj >= 0 && zk >= 0 && xi <= n && yj <= n && zk <= n;
    const int64_t oc = o0 + dx + dy * g.px + dz * g.py;
    if (PRED) {
      nb[o][0] = nb[o][1] = nb[o][2] = 0.0;
      nb[o][3] = (in && !((xi + yj + zk) & 1)) ? __ldg(Pf + oc) : 0.0;
    } else {
      const unsigned em = in ? elim_mask(dm, g.slipmask, n, xi, yj, zk) : 7u;
#pragma unroll
      for (int f = 0; f < 3; ++f) nb[o][f] = ((em >> f) & 1u) ? 0.0 : __ldg(U + f * g.fs + oc);
      nb[o][3] = in ? __ldg(Pf + oc) : 0.0;
    }
  }
  // classes of the star tets (cube own, tet t): 0xFF outside the cube
  uint8_t cls[8][6];
#pragma unroll
  for (int own = 0; own < 8; ++own) {
    const int ci = i - (own & 1), cj = j - ((own >> 1) & 1), ck = k - (own >> 2);
    const bool in = ci >= 0 && cj >= 0 && ck >= 0 && ci < n && cj < n && ck < n;
    const uint8_t* clp = g.cls + ((((int64_t)(ck - g.cz0)) * n + cj) * n + ci) * 6;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      if (kcorner(own, t) < 0) continue;
      cls[own][t] = in ? __ldg(clp + t) : (uint8_t)0xFF;
    }
  }
  y[0] = y[1] = y[2] = y[3] = 0.0;
  dA[0] = dA[1] = dA[2] = 0.0;
  dC = 0.0;
#pragma unroll
  for (int own = 0; own < 8; ++own) {
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const int m = kcorner(own, t);
      if (m < 0) continue;
      const int cl = cls[own][t];
      if (cl == 0xFF) continue;
      const int s1 = kperm(t, 0), s2 = kperm(t, 1), s3 = kperm(t, 2);
      // neighbourhood index of tet vertex q: cube corner c relative to the vertex
      auto vo = [&](int q) {
        const int c = ktet_corner(t, q);
        const int dx = (c & 1) - (own & 1), dy = ((c >> 1) & 1) - ((own >> 1) & 1), dz = (c >> 2) - (own >> 2);
        return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
      };
      const int v0 = vo(0), v1 = vo(1), v2 = vo(2), v3 = vo(3);
      double G[3][3], gp[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        G[a][s1] = (nb[v1][a] - nb[v0][a]) * hinv;
        G[a][s2] = (nb[v2][a] - nb[v1][a]) * hinv;
        G[a][s3] = (nb[v3][a] - nb[v2][a]) * hinv;
      }
      gp[s1] = (nb[v1][3] - nb[v0][3]) * hinv;
      gp[s2] = (nb[v2][3] - nb[v1][3]) * hinv;
      gp[s3] = (nb[v3][3] - nb[v2][3]) * hinv;
      double gm[3] = {0.0, 0.0, 0.0};
      if (m == 0) {
        gm[s1] = -hinv;
      } else if (m == 1) {
        gm[s1] = hinv; gm[s2] = -hinv;
      } else if (m == 2) {
        gm[s2] = hinv; gm[s3] = -hinv;
      } else {
        gm[s3] = hinv;
      }
      double mu, imu;
      tet_coef(g, i - (own & 1), j - ((own >> 1) & 1), k - (own >> 2), t, cl, mu, imu);
      const double gg = gm[0] * gm[0] + gm[1] * gm[1] + gm[2] * gm[2];
      const double tr = G[0][0] + G[1][1] + G[2][2];
      if (blocks & BLK_A) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double s = G[a][0] * gm[0] + G[a][1] * gm[1] + G[a][2] * gm[2];
          if (FORM != FORM_GRAD) s += G[0][a] * gm[0] + G[1][a] * gm[1] + G[2][a] * gm[2];
          if (FORM == FORM_MOD) s -= tr * gm[a];
          y[a] += mu * vol * s;
        }
      }
      if (blocks & BLK_BT) {
        const double ps = nb[v0][3] + nb[v1][3] + nb[v2][3] + nb[v3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) y[a] -= vq * gm[a] * ps;
      }
      if (blocks & BLK_B) y[3] -= vq * tr;
      if (blocks & BLK_C) y[3] -= cstab * imu * (gm[0] * gp[0] + gm[1] * gp[1] + gm[2] * gp[2]);
#pragma unroll
      for (int a = 0; a < 3; ++a)
        dA[a] += mu * vol * (gg + (FORM == FORM_SYM ? gm[a] * gm[a] : 0.0));
      dC += cstab * imu * gg;
    }
  }
  {
    const unsigned em = elim(g, i, j, k);
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if ((em >> a) & 1u) y[a] = 0.0;
  }
}

// w_j = int phi_j / mu = sum_{T ni j} |T| / (4 mu_T)   (gauge weight)
__device__ __forceinline__ double gauge_weight(const DGrid& g, int i, int j, int k) {
  const double vq = 0.25 * g.h * g.h * g.h / 6.0;
  double w = 0.0;
  for (int dz = -1; dz <= 0; ++dz) {
    const int ck = k + dz;
    if (ck < 0 || ck >= g.n) continue;
    for (int dy = -1; dy <= 0; ++dy) {
      const int cj = j + dy;
      if (cj < 0 || cj >= g.n) continue;
      for (int dx = -1; dx <= 0; ++dx) {
        const int ci = i + dx;
        if (ci < 0 || ci >= g.n) continue;
        const int corner = (-dx) | ((-dy) << 1) | ((-dz) << 2);
        for (int t = 0; t < 6; ++t)
          if (c_corner_m[corner][t] >= 0) {
            double mu, imu;
            tet_coef(g, ci, cj, ck, t, elem_class(g, ci, cj, ck, t), mu, imu);
            w += vq * imu;
          }
      }
    }
  }
  return w;
}

// the 15 Kuhn offsets (0, +-d, d in {0,1}^3 \ 0) as 27-point indices
__host__ __device__ constexpr int kq_dx(int q) { return q == 0 ? 0 : (q & 1 ? 1 : -1) * (((q - 1) / 2 + 1) & 1); }
__host__ __device__ constexpr int kq_dy(int q) { return q == 0 ? 0 : (q & 1 ? 1 : -1) * ((((q - 1) / 2 + 1) >> 1) & 1); }
__host__ __device__ constexpr int kq_dz(int q) { return q == 0 ? 0 : (q & 1 ? 1 : -1) * ((((q - 1) / 2 + 1) >> 2) & 1); }
constexpr int NQ = 15;
constexpr bool kq_table_ok() {
  // the 15 offsets are distinct and exactly the Kuhn pattern
  int seen[27] = {};
  for (int q = 0; q < NQ; ++q) {
    const int dx = kq_dx(q), dy = kq_dy(q), dz = kq_dz(q);
    if (!((dx >= 0 && dy >= 0 && dz >= 0) || (dx <= 0 && dy <= 0 && dz <= 0))) return false;
    const int o = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
    if (seen[o]++) return false;
  }
  return true;
}
static_assert(kq_table_ok(), "Kuhn offset table");

// explicit stencil of a row: S[r][q][c] (r, c: u1,u2,u3,p), the entries of K,
// then the inverse diagonals 1/A_00, 1/A_11, 1/A_22, 1/C (Gauss-Seidel)
constexpr int EXPL = 4 * NQ * 4 + 4;

__device__ __forceinline__ int qoff(const DGrid& g, int q) {
  return kq_dx(q) + kq_dy(q) * (int)g.px + kq_dz(q) * (int)g.py;
}

// colour-1 vertex: its colour-0 Kuhn neighbours are those at an odd offset sum
__device__ __forceinline__ constexpr bool q_odd(int q) { return ((kq_dx(q) + kq_dy(q) + kq_dz(q)) & 1) != 0; }

}  // namespace stk
