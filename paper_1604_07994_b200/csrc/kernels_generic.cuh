// Generic (element-row) kernels: one thread per owned vertex, every row by
// the element loop (row_list: neighbourhood gathered up front).  Used on the small levels (n < 64) and as
// the reference device path for the tiled constant-stencil kernels.
#pragma once
#include "stk_common.cuh"

namespace stk {

__device__ __forceinline__ bool owned_vertex(const DGrid& g, int64_t t, int& i, int& j, int& k) {
  const int64_t nx = g.n + 1;
  const int64_t per = nx * nx;
  if (t >= per * g.nzl) return false;
  k = g.z0 + (int)(t / per);
  const int64_t r = t % per;
  j = (int)(r / nx);
  i = (int)(r % nx);
  return true;
}

template <int FORM>
__global__ void k_apply_generic(DGrid g, const double* __restrict__ x, double* __restrict__ y,
                                unsigned blocks) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  double r[4], dA[3], dC;
  row_list<FORM, false>(g, i, j, k, x, x + 3 * g.fs, blocks, r, dA, dC);
  const int64_t o = vidx(g, i, j, k);
#pragma unroll
  for (int f = 0; f < 4; ++f) y[f * g.fs + o] = r[f];
}

// r = b - K x  (velocity rows 0 at Dirichlet vertices)
template <int FORM>
__global__ void k_residual_generic(DGrid g, const double* __restrict__ x,
                                   const double* __restrict__ b, double* __restrict__ r) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  double y[4], dA[3], dC;
  row_list<FORM, false>(g, i, j, k, x, x + 3 * g.fs, BLK_ALL, y, dA, dC);
  const int64_t o = vidx(g, i, j, k);
  const unsigned em = elim(g, i, j, k);
#pragma unroll
  for (int f = 0; f < 4; ++f) r[f * g.fs + o] = ((em >> f) & 1u) ? 0.0 : b[f * g.fs + o] - y[f];
}

// One colour pass of the velocity Gauss-Seidel (Jacobi within the colour):
//   u_out = u_in + (f - A u_in - B^T p) / diag(A)  at vertices of colour `color`
//   u_out = u_in                                  elsewhere
template <int FORM>
__global__ void k_vel_pass_generic(DGrid g, const double* __restrict__ uin,
                                   const double* __restrict__ p, const double* __restrict__ b,
                                   double* __restrict__ uout, int color, int ncolors) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const int64_t o = vidx(g, i, j, k);
  const unsigned em = elim(g, i, j, k);
  const bool active = ((i + j + k) % ncolors == color) && em != 7u;
  if (!active) {
#pragma unroll
    for (int a = 0; a < 3; ++a) uout[a * g.fs + o] = ((em >> a) & 1u) ? 0.0 : uin[a * g.fs + o];
    return;
  }
  double y[4], dA[3], dC;
  row_list<FORM, false>(g, i, j, k, uin, p, BLK_A | BLK_BT, y, dA, dC);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    uout[a * g.fs + o] = ((em >> a) & 1u) ? 0.0 : uin[a * g.fs + o] + (b[a * g.fs + o] - y[a]) / dA[a];
}

// Pressure step, part 1:  r_p = B u - C p - g ;  T = r_p / C_ii (colour 0), r_p (colour 1)
template <int FORM>
__global__ void k_p_pass1_generic(DGrid g, const double* __restrict__ x,
                                  const double* __restrict__ gp, double* __restrict__ T) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  double y[4], dA[3], dC;
  row_list<FORM, false>(g, i, j, k, x, x + 3 * g.fs, BLK_B | BLK_C, y, dA, dC);
  const int64_t o = vidx(g, i, j, k);
  const double r = y[3] - gp[o];
  T[o] = ((i + j + k) & 1) == 0 ? r / dC : r;
}

// Pressure step, part 2: delta_1 = (r_p - C delta_0)/C_ii on colour 1,
// delta_0 = T on colour 0;  p += omega * delta
template <int FORM>
__global__ void k_p_pass2_generic(DGrid g, const double* __restrict__ T, double* __restrict__ p,
                                  double omega) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const int64_t o = vidx(g, i, j, k);
  double d;
  if (((i + j + k) & 1) == 0) {
    d = T[o];
  } else {
    double y[4], dA[3], dC;
    row_list<FORM, true>(g, i, j, k, nullptr, T, BLK_C, y, dA, dC);
    d = (T[o] + y[3]) / dC;   // y[3] = -(C delta_0)_i
  }
  p[o] += omega * d;
}

// b_c = P^T r_f: (R r)(I) = r(2I) + 1/2 sum_{d in +-D+} r(2I + d)   (DESIGN R14)
__global__ void k_restrict(DGrid gf, DGrid gc, const double* __restrict__ rf,
                           double* __restrict__ bc) {
  int I, J, K;
  if (!owned_vertex(gc, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, I, J, K)) return;
  const int fi = 2 * I, fj = 2 * J, fk = 2 * K;
  const int D[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};
  const unsigned em = elim(gc, I, J, K);
  const int64_t oc = vidx(gc, I, J, K);
  for (int f = 0; f < 4; ++f) {
    if ((em >> f) & 1u) { bc[f * gc.fs + oc] = 0.0; continue; }
    const double* r = rf + f * gf.fs;
    double s = r[vidx(gf, fi, fj, fk)];
    double e = 0.0;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      for (int sg = -1; sg <= 1; sg += 2) {
        const int a = fi + sg * D[q][0], b = fj + sg * D[q][1], c = fk + sg * D[q][2];
        if (a < 0 || b < 0 || c < 0 || a > gf.n || b > gf.n || c > gf.n) continue;
        e += r[vidx(gf, a, b, c)];
      }
    }
    bc[f * gc.fs + oc] = s + 0.5 * e;
  }
}

// x_f += P x_c: fine vertex 2I + d (d in {0,1}^3) takes x_c(I) (d = 0) or the
// mean of the coarse Kuhn edge (I, I + d)
__global__ void k_prolong_add(DGrid gc, DGrid gf, const double* __restrict__ xc,
                              double* __restrict__ xf) {
  int i, j, k;
  if (!owned_vertex(gf, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const int64_t of = vidx(gf, i, j, k);
  const unsigned em = elim(gf, i, j, k);
  const int I = i >> 1, J = j >> 1, K = k >> 1;
  const int di = i & 1, dj = j & 1, dk = k & 1;
  const int64_t o0 = vidx(gc, I, J, K);
  const bool mid = di | dj | dk;
  const int64_t o1 = mid ? vidx(gc, I + di, J + dj, K + dk) : o0;
  for (int f = 0; f < 4; ++f) {
    if ((em >> f) & 1u) { xf[f * gf.fs + of] = 0.0; continue; }
    const double v = mid ? 0.5 * (xc[f * gc.fs + o0] + xc[f * gc.fs + o1]) : xc[f * gc.fs + o0];
    xf[f * gf.fs + of] += v;
  }
}

// per-block partial sums for the squared norms (velocity masked) and the
// gauge sums: out[block][0..3] = sum x_f^2, [4] = sum w p, [5] = sum w
__global__ void k_partials(DGrid g, const double* __restrict__ x, double* __restrict__ part,
                           int with_gauge) {
  __shared__ double sh[6][256];
  int i, j, k;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       owned_vertex(g, t, i, j, k); t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = vidx(g, i, j, k);
    const unsigned em = elim(g, i, j, k);
    for (int f = 0; f < 4; ++f) {
      const double v = ((em >> f) & 1u) ? 0.0 : x[f * g.fs + o];
      acc[f] += v * v;
    }
    if (with_gauge) {
      const double w = gauge_weight(g, i, j, k);
      acc[4] += w * x[3 * g.fs + o];
      acc[5] += w;
    }
  }
  for (int q = 0; q < 6; ++q) sh[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int q = 0; q < 6; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) part[blockIdx.x * 6 + q] = sh[q][0];
}

// fixed-order final sum of the partials (deterministic)
__global__ void k_partials_final(const double* __restrict__ part, int nblocks,
                                 double* __restrict__ out) {
  __shared__ double sh[6][256];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
    for (int q = 0; q < 6; ++q) acc[q] += part[b * 6 + q];
  for (int q = 0; q < 6; ++q) sh[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int q = 0; q < 6; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) out[q] = sh[q][0];
}

// p -= (sum w p)/(sum w), sums read from device memory
__global__ void k_gauge_apply(DGrid g, double* __restrict__ x, const double* __restrict__ sums) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const double mean = sums[4] / sums[5];
  x[3 * g.fs + vidx(g, i, j, k)] -= mean;
}

// nodal forcing: b_u = M f  (consistent mass, (phi_i,phi_j)_T = |T|/20 (1 + delta_ij)),
// f in the padded level layout (fields 0..2, halo planes valid); b_p = 0; Dirichlet rows 0
__global__ void k_load_nodal(DGrid g, const double* __restrict__ f, double* __restrict__ b) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const double c = g.h * g.h * g.h / 6.0 / 20.0;
  double acc[3] = {0, 0, 0};
  auto fval = [&](int a, int ii, int jj, int kk) -> double { return f[a * g.fs + vidx(g, ii, jj, kk)]; };
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
        for (int t = 0; t < 6; ++t) {
          if (c_corner_m[corner][t] < 0) continue;
          const int s1 = c_perm[t][0], s2 = c_perm[t][1];
          int v1[3] = {ci, cj, ck}; v1[s1] += 1;
          int v2[3] = {v1[0], v1[1], v1[2]}; v2[s2] += 1;
          for (int a = 0; a < 3; ++a) {
            const double sum = fval(a, ci, cj, ck) + fval(a, v1[0], v1[1], v1[2]) +
                               fval(a, v2[0], v2[1], v2[2]) + fval(a, ci + 1, cj + 1, ck + 1);
            acc[a] += c * (sum + fval(a, i, j, k));
          }
        }
      }
    }
  }
  const int64_t o = vidx(g, i, j, k);
  const unsigned em = elim(g, i, j, k);
  for (int a = 0; a < 3; ++a) b[a * g.fs + o] = ((em >> a) & 1u) ? 0.0 : acc[a];
  b[3 * g.fs + o] = 0.0;
}

// element-constant forcing: b_{i,a} = sum_T f_{T,a} |T| / 4 ; fcls per element (same
// layout as the viscosity classes), table [3 * nftab] in device memory
__global__ void k_load_elem(DGrid g, const uint8_t* __restrict__ fcls,
                            const double* __restrict__ table, double* __restrict__ b) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const double vq = 0.25 * g.h * g.h * g.h / 6.0;
  double acc[3] = {0, 0, 0};
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
        for (int t = 0; t < 6; ++t) {
          if (c_corner_m[corner][t] < 0) continue;
          const uint8_t fc = fcls[((((int64_t)(ck - g.cz0)) * g.n + cj) * g.n + ci) * 6 + t];
          for (int a = 0; a < 3; ++a) acc[a] += vq * table[3 * fc + a];
        }
      }
    }
  }
  const int64_t o = vidx(g, i, j, k);
  const unsigned em = elim(g, i, j, k);
  for (int a = 0; a < 3; ++a) b[a * g.fs + o] = ((em >> a) & 1u) ? 0.0 : acc[a];
  b[3 * g.fs + o] = 0.0;
}

// canonical (4 x (n+1)^2 x nzl, field-major) <-> padded layout
__global__ void k_pack(DGrid g, const double* __restrict__ canon, double* __restrict__ dev,
                       int nfields) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const int64_t nx = g.n + 1, per = nx * nx, cs = per * g.nzl;
  const int64_t c = (int64_t)(k - g.z0) * per + (int64_t)j * nx + i;
  const int64_t o = vidx(g, i, j, k);
  for (int f = 0; f < nfields; ++f) dev[f * g.fs + o] = canon[f * cs + c];
}
__global__ void k_iota(int32_t* __restrict__ a, int64_t n) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) a[t] = (int32_t)t;
}

// velocity entries of eliminated DoFs (Dirichlet faces, free-slip normals) set to 0
__global__ void k_zero_eliminated(DGrid g, double* __restrict__ v) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const unsigned em = elim(g, i, j, k);
  if (!em) return;
  const int64_t o = vidx(g, i, j, k);
  for (int a = 0; a < 3; ++a)
    if ((em >> a) & 1u) v[a * g.fs + o] = 0.0;
}
__global__ void k_unpack(DGrid g, const double* __restrict__ dev, double* __restrict__ canon) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const int64_t nx = g.n + 1, per = nx * nx, cs = per * g.nzl;
  const int64_t c = (int64_t)(k - g.z0) * per + (int64_t)j * nx + i;
  const int64_t o = vidx(g, i, j, k);
  for (int f = 0; f < 4; ++f) canon[f * cs + c] = dev[f * g.fs + o];
}

// ---- setup kernels -------------------------------------------------------

// coarse element coefficients of cube layers [CK0, CK1) (reading R15): for the 8 Bey
// children of each coarse tet, mu_A = arithmetic mean of the children's
// mu_A (the rediscretised coarse A is then the Galerkin product P^T A P), 1/mu_C = mean
// of the children's 1/mu_C; the class is the children's common class, else CLS_MIXED.
// gf/gc: fine/coarse grids (cube layers stored); cls_c / emu_c in gc's layout.
__global__ void k_coarsen(DGrid gf, DGrid gc, int CK0, int CK1, uint8_t* __restrict__ cls_c,
                          double2* __restrict__ emu_c, int harmonic) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int nc = gc.n;
  const int64_t total = (int64_t)(CK1 - CK0) * nc * nc * 6;
  if (tid >= total) return;
  const int T = (int)(tid % 6);
  int64_t r = tid / 6;
  const int CI = (int)(r % nc);
  r /= nc;
  const int CJ = (int)(r % nc);
  const int CK = CK0 + (int)(r / nc);
  double sm = 0.0, si = 0.0;
  int c0 = -1;
  bool pure = true;
  for (int q = 0; q < 8; ++q) {
    const int off = c_child_off[T][q];
    const int fi = 2 * CI + (off & 1), fj = 2 * CJ + ((off >> 1) & 1), fk = 2 * CK + ((off >> 2) & 1);
    const int ft = c_child_t[T][q];
    const int cl = elem_class(gf, fi, fj, fk, ft);
    double mu, imu;
    tet_coef(gf, fi, fj, fk, ft, cl, mu, imu);
    sm += harmonic ? 1.0 / mu : mu;
    si += imu;
    if (q == 0) c0 = cl;
    pure = pure && cl == c0 && cl != CLS_MIXED;
  }
  const int64_t o = elem_index(gc, CI, CJ, CK, T);
  cls_c[o] = pure ? (uint8_t)c0 : CLS_MIXED;
  // mu_A: arithmetic mean of the 8 children (R15; the Galerkin product), or harmonic
  // (coarse_mu = 2); 1/mu_C: arithmetic mean of the children's 1/mu_C
  emu_c[o] = make_double2(harmonic ? 8.0 / sm : sm * 0.125, si * 0.125);
}

// number of entries >= lim (input validation of the element classes)
__global__ void k_count_ge(const uint8_t* __restrict__ a, int64_t n, int lim, unsigned long long* cnt) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n && a[t] >= lim) atomicAdd(cnt, 1ull);
}

// per-vertex code (R6): class k (< 0x40) when
// the star of tets inside the cube is isoviscous with class k AND the vertex is
// interior or lies only on Dirichlet faces (then its velocity rows are
// eliminated and its pressure row is the truncated constant stencil);
// 0x40 | k for an isoviscous vertex of the traction top face z = 1 that lies on
// no other face (truncated constant stencils of the 4 cubes below); else
// CODE_IRREGULAR (Gamma_12, other Gamma_F rows, classes >= 0x40): a list row
// evaluated by the element loop.  Counts list rows into *nirr.
__global__ void k_classify(DGrid g, uint8_t* __restrict__ code, unsigned long long* nirr) {
  int i, j, k;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (!owned_vertex(g, tid, i, j, k)) return;
  uint8_t c = CODE_IRREGULAR;
  const unsigned m = g.dirmask;
  const bool faces_ok = (i > 0 || (m & 1u)) && (i < g.n || (m & 2u)) && (j > 0 || (m & 4u)) &&
                        (j < g.n || (m & 8u)) && (k > 0 || (m & 16u)) && (k < g.n || (m & 32u));
  // a vertex on the traction top face z = 1 and on no other face (Gamma_F)
  const bool top = k == g.n && !(m & 32u) && !(g.slipmask & 32u) && i > 0 && i < g.n && j > 0 && j < g.n;
  if (faces_ok || top) {
    bool same = true;
    int first = -1;
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
          for (int t = 0; t < 6; ++t) {
            if (c_corner_m[corner][t] < 0) continue;
            const int cl = elem_class(g, ci, cj, ck, t);
            if (cl == CLS_MIXED) same = false;  // coarse tet of several classes: never regular (R15)
            if (first < 0) first = cl;
            else if (cl != first && mu_of(g, cl) != mu_of(g, first)) same = false;
          }
        }
      }
    }
    if (same && first >= 0) {
      if (top) {
        if (first < 0x40) c = (uint8_t)(0x40 | first);   // CODE_TOP | class
      } else if (first < 0x40) {
        c = (uint8_t)first;
      }
    }
  }
  code[vidx(g, i, j, k)] = c;
  if (c == CODE_IRREGULAR) atomicAdd(nirr, 1ull);
}

// compact list of the owned list rows (CODE_IRREGULAR), as owned linear indices
// t = (k - z0) (n+1)^2 + j (n+1) + i; *cnt must be zeroed.  Order is irrelevant:
// every row is evaluated independently.
// (top = 1: instead the isoviscous traction-face rows, code 0x40 | k -- the rows whose
// truncated stencils couple within a colour, for the repeat pass of the smoother)
__global__ void k_build_list(DGrid g, int32_t* __restrict__ list, unsigned long long* cnt, int top = 0) {
  int i, j, k;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (!owned_vertex(g, tid, i, j, k)) return;
  const uint8_t c = g.code[vidx(g, i, j, k)];
  const bool take = top ? (c >= 0x40 && c != CODE_IRREGULAR) : c == CODE_IRREGULAR;
  if (take) list[atomicAdd(cnt, 1ull)] = (int32_t)tid;
}
__global__ void k_count_top(DGrid g, unsigned long long* cnt) {
  int i, j, k;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (!owned_vertex(g, tid, i, j, k)) return;
  const uint8_t c = g.code[vidx(g, i, j, k)];
  if (c >= 0x40 && c != CODE_IRREGULAR) atomicAdd(cnt, 1ull);
}

// ---- coarsest level: dense assembly, Gauss-Jordan inverse, apply -----------

struct FetchUnit {
  int ui, uj, uk, uf;
  __device__ __forceinline__ double operator()(const DGrid& g, int i, int j, int k, int f) const {
    return (i == ui && j == uj && k == uk && f == uf) ? 1.0 : 0.0;
  }
};

// K[r][c] = row r of K applied to the unit vector of free DoF c; N1 = leading dim.
// dofs[q] = (f << 28) | (k << 18) | (j << 9) | i  (global coordinates)
template <int FORM>
__global__ void k_coarse_assemble(DGrid g, const int32_t* __restrict__ dofs, int N, int N1,
                                  double* __restrict__ K, int gauge) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= (int64_t)N1 * N1) return;
  const int r = (int)(tid / N1), c = (int)(tid % N1);
  double v = 0.0;
  auto unpack = [](int32_t d, int& f, int& i, int& j, int& k) {
    f = (d >> 28) & 0xF; k = (d >> 18) & 0x3FF; j = (d >> 9) & 0x1FF; i = d & 0x1FF;
  };
  if (r < N && c < N) {
    int fr, ir, jr, kr, fc, ic, jc, kc;
    unpack(dofs[r], fr, ir, jr, kr);
    unpack(dofs[c], fc, ic, jc, kc);
    if (abs(ir - ic) <= 1 && abs(jr - jc) <= 1 && abs(kr - kc) <= 1) {
      FetchUnit fx{ic, jc, kc, fc};
      double y[4], dA[3], dC;
      row_generic<FORM>(g, ir, jr, kr, fx, BLK_ALL, y, dA, dC);
      v = y[fr];
    }
  } else if (gauge && (r < N || c < N) && !(r == N && c == N)) {
    const int q = r < N ? r : c;
    int f, i, j, k;
    unpack(dofs[q], f, i, j, k);
    v = f == 3 ? gauge_weight(g, i, j, k) : 0.0;
  }
  K[(int64_t)r * N1 + c] = v;
}


// x_F = G b_F on the coarsest level (G: N x N with leading dimension ld); other entries 0
__global__ void k_coarse_apply(DGrid g, const int32_t* __restrict__ dofs, int N, int ld,
                               const double* __restrict__ G, const double* __restrict__ b,
                               double* __restrict__ x) {
  extern __shared__ double bs[];
  for (int q = threadIdx.x; q < N; q += blockDim.x) {
    const int32_t d = dofs[q];
    const int f = (d >> 28) & 0xF, k = (d >> 18) & 0x3FF, j = (d >> 9) & 0x1FF, i = d & 0x1FF;
    bs[q] = b[f * g.fs + vidx(g, i, j, k)];
  }
  __syncthreads();
  // zero everything first (Dirichlet entries), then write free entries
  const int64_t nx = g.n + 1;
  for (int64_t e = threadIdx.x; e < nx * nx * g.nzl; e += blockDim.x) {
    const int i = (int)(e % nx), j = (int)((e / nx) % nx), k = g.z0 + (int)(e / (nx * nx));
    for (int f = 0; f < 4; ++f) x[f * g.fs + vidx(g, i, j, k)] = 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < N; r += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < N; ++c) s += G[(int64_t)r * ld + c] * bs[c];
    const int32_t d = dofs[r];
    const int f = (d >> 28) & 0xF, k = (d >> 18) & 0x3FF, j = (d >> 9) & 0x1FF, i = d & 0x1FF;
    x[f * g.fs + vidx(g, i, j, k)] = s;
  }
}


// ---- warp-per-row kernels for the small levels (n <= 32) --------------------
// With few rows per level the kernel time is the latency of one row, so a row
// is spread over a warp: lane l < 24 integrates tet l of the star.

// star tets of a vertex, lane -> own corner | tet << 3 (own corners 0..7 in
// order, tets 0..5 in order), packed 6 bits per lane at compile time
__host__ __device__ constexpr int kstar_entry(int l) {
  int cnt = 0;
  for (int own = 0; own < 8; ++own)
    for (int t = 0; t < 6; ++t)
      if (kcorner(own, t) >= 0) {
        if (cnt == l) return own | (t << 3);
        ++cnt;
      }
  return 0;
}
__host__ __device__ constexpr uint64_t kstar_pack(int w) {
  uint64_t v = 0;
  for (int q = 0; q < 8; ++q) v |= (uint64_t)kstar_entry(8 * w + q) << (8 * q);
  return v;
}
constexpr uint64_t KSTAR0 = kstar_pack(0), KSTAR1 = kstar_pack(1), KSTAR2 = kstar_pack(2);
static_assert(kstar_entry(23) == (7 | (5 << 3)), "24 star tets");

// The row of row_generic at (i,j,k), one warp: lane l < 24 integrates star tet
// l from global memory, a butterfly reduction gives all lanes y[4], dA[3], dC.
template <int FORM, bool PRED>
__device__ __forceinline__ void row_warp(const DGrid& g, int i, int j, int k, const double* __restrict__ U,
                                         const double* __restrict__ Pf, unsigned blocks, double y[4], double dA[3],
                                         double& dC) {
  const int lane = threadIdx.x & 31;
  double r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int n = g.n;
  if (lane < 24) {
    const uint64_t w = lane < 8 ? KSTAR0 : lane < 16 ? KSTAR1 : KSTAR2;
    const int e = (int)((w >> (8 * (lane & 7))) & 0xFF);
    const int own = e & 7, t = e >> 3;
    const int ci = i - (own & 1), cj = j - ((own >> 1) & 1), ck = k - (own >> 2);
    if (ci >= 0 && cj >= 0 && ck >= 0 && ci < n && cj < n && ck < n) {
      const double h = g.h, hinv = 1.0 / h;
      const double vol = h * h * h / 6.0, vq = 0.25 * vol;
      const double cstab = g.delta * h * h * vol;
      const unsigned dm = g.dirmask;
      const int s1 = kperm(t, 0), s2 = kperm(t, 1), s3 = kperm(t, 2);
      const int m = kcorner(own, t);
      const int cl = g.cls[((((int64_t)(ck - g.cz0)) * n + cj) * n + ci) * 6 + t];
      double val[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = ktet_corner(t, q);
        const int xi = ci + (c & 1), yj = cj + ((c >> 1) & 1), zk = ck + (c >> 2);
        const int64_t oc = vidx(g, xi, yj, zk);
        if (PRED) {
          val[q][0] = val[q][1] = val[q][2] = 0.0;
          val[q][3] = ((xi + yj + zk) & 1) ? 0.0 : __ldg(Pf + oc);
        } else {
          const unsigned em = elim_mask(dm, g.slipmask, n, xi, yj, zk);
#pragma unroll
          for (int f = 0; f < 3; ++f) val[q][f] = ((em >> f) & 1u) ? 0.0 : __ldg(U + f * g.fs + oc);
          val[q][3] = __ldg(Pf + oc);
        }
      }
      double G[3][3], gp[3], gm[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double d1 = (val[1][a] - val[0][a]) * hinv, d2 = (val[2][a] - val[1][a]) * hinv,
                     d3 = (val[3][a] - val[2][a]) * hinv;
        G[a][0] = s1 == 0 ? d1 : s2 == 0 ? d2 : d3;
        G[a][1] = s1 == 1 ? d1 : s2 == 1 ? d2 : d3;
        G[a][2] = s1 == 2 ? d1 : s2 == 2 ? d2 : d3;
      }
      {
        const double d1 = (val[1][3] - val[0][3]) * hinv, d2 = (val[2][3] - val[1][3]) * hinv,
                     d3 = (val[3][3] - val[2][3]) * hinv;
        gp[0] = s1 == 0 ? d1 : s2 == 0 ? d2 : d3;
        gp[1] = s1 == 1 ? d1 : s2 == 1 ? d2 : d3;
        gp[2] = s1 == 2 ? d1 : s2 == 2 ? d2 : d3;
      }
      // grad lambda_m: -e_s1 (m=0), e_s1 - e_s2 (1), e_s2 - e_s3 (2), e_s3 (3), over h
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double v;
        if (m == 0) v = (d == s1) ? -hinv : 0.0;
        else if (m == 1) v = (d == s1) ? hinv : (d == s2) ? -hinv : 0.0;
        else if (m == 2) v = (d == s2) ? hinv : (d == s3) ? -hinv : 0.0;
        else v = (d == s3) ? hinv : 0.0;
        gm[d] = v;
      }
      double mu, imu;
      tet_coef(g, ci, cj, ck, t, cl, mu, imu);
      const double gg = gm[0] * gm[0] + gm[1] * gm[1] + gm[2] * gm[2];
      const double tr = G[0][0] + G[1][1] + G[2][2];
      if (blocks & BLK_A) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double sv = G[a][0] * gm[0] + G[a][1] * gm[1] + G[a][2] * gm[2];
          if (FORM != FORM_GRAD) sv += G[0][a] * gm[0] + G[1][a] * gm[1] + G[2][a] * gm[2];
          if (FORM == FORM_MOD) sv -= tr * gm[a];
          r[a] += mu * vol * sv;
        }
      }
      if (blocks & BLK_BT) {
        const double ps = val[0][3] + val[1][3] + val[2][3] + val[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) r[a] -= vq * gm[a] * ps;
      }
      if (blocks & BLK_B) r[3] -= vq * tr;
      if (blocks & BLK_C) r[3] -= cstab * imu * (gm[0] * gp[0] + gm[1] * gp[1] + gm[2] * gp[2]);
#pragma unroll
      for (int a = 0; a < 3; ++a) r[4 + a] = mu * vol * (gg + (FORM == FORM_SYM ? gm[a] * gm[a] : 0.0));
      r[7] = cstab * imu * gg;
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] += __shfl_xor_sync(0xffffffffu, r[q], off);
  y[0] = r[0]; y[1] = r[1]; y[2] = r[2]; y[3] = r[3];
  dA[0] = r[4]; dA[1] = r[5]; dA[2] = r[6];
  dC = r[7];
  const unsigned em = elim(g, i, j, k);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if ((em >> a) & 1u) y[a] = 0.0;
}

constexpr int GW_NT = 128;  // 4 rows per CTA
__device__ __forceinline__ bool warp_vertex(const DGrid& g, int& i, int& j, int& k) {
  return owned_vertex(g, (blockIdx.x * (int64_t)GW_NT + threadIdx.x) >> 5, i, j, k);
}

template <int FORM>
__global__ void __launch_bounds__(GW_NT) k_apply_gw(DGrid g, const double* __restrict__ x, double* __restrict__ y,
                                                    unsigned blocks) {
  int i, j, k;
  if (!warp_vertex(g, i, j, k)) return;
  double r[4], dA[3], dC;
  row_warp<FORM, false>(g, i, j, k, x, x + 3 * g.fs, blocks, r, dA, dC);
  if ((threadIdx.x & 31) == 0) {
    const int64_t o = vidx(g, i, j, k);
#pragma unroll
    for (int f = 0; f < 4; ++f) y[f * g.fs + o] = r[f];
  }
}

template <int FORM>
__global__ void __launch_bounds__(GW_NT) k_residual_gw(DGrid g, const double* __restrict__ x,
                                                       const double* __restrict__ b, double* __restrict__ r) {
  int i, j, k;
  if (!warp_vertex(g, i, j, k)) return;
  double y[4], dA[3], dC;
  row_warp<FORM, false>(g, i, j, k, x, x + 3 * g.fs, BLK_ALL, y, dA, dC);
  if ((threadIdx.x & 31) == 0) {
    const int64_t o = vidx(g, i, j, k);
    const unsigned em = elim(g, i, j, k);
#pragma unroll
    for (int f = 0; f < 4; ++f) r[f * g.fs + o] = ((em >> f) & 1u) ? 0.0 : b[f * g.fs + o] - y[f];
  }
}

template <int FORM>
__global__ void __launch_bounds__(GW_NT) k_vel_pass_gw(DGrid g, const double* __restrict__ uin,
                                                       const double* __restrict__ p, const double* __restrict__ b,
                                                       double* __restrict__ uout, int color, int ncolors) {
  int i, j, k;
  if (!warp_vertex(g, i, j, k)) return;
  const int64_t o = vidx(g, i, j, k);
  const unsigned em = elim(g, i, j, k);
  const bool active = ((i + j + k) % ncolors == color) && em != 7u;  // warp-uniform
  double y[4], dA[3], dC;
  if (active) row_warp<FORM, false>(g, i, j, k, uin, p, BLK_A | BLK_BT, y, dA, dC);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
      uout[a * g.fs + o] = ((em >> a) & 1u) ? 0.0
                           : active        ? uin[a * g.fs + o] + (b[a * g.fs + o] - y[a]) / dA[a]
                                           : uin[a * g.fs + o];
  }
}

template <int FORM>
__global__ void __launch_bounds__(GW_NT) k_p_pass1_gw(DGrid g, const double* __restrict__ x,
                                                      const double* __restrict__ gp, double* __restrict__ T) {
  int i, j, k;
  if (!warp_vertex(g, i, j, k)) return;
  double y[4], dA[3], dC;
  row_warp<FORM, false>(g, i, j, k, x, x + 3 * g.fs, BLK_B | BLK_C, y, dA, dC);
  if ((threadIdx.x & 31) == 0) {
    const int64_t o = vidx(g, i, j, k);
    const double r = y[3] - gp[o];
    T[o] = ((i + j + k) & 1) == 0 ? r / dC : r;
  }
}

template <int FORM>
__global__ void __launch_bounds__(GW_NT) k_p_pass2_gw(DGrid g, const double* __restrict__ T, double* __restrict__ p,
                                                      double omega) {
  int i, j, k;
  if (!warp_vertex(g, i, j, k)) return;
  const int64_t o = vidx(g, i, j, k);
  double d = 0.0;
  if (((i + j + k) & 1) == 0) {
    d = T[o];
  } else {
    double y[4], dA[3], dC;
    row_warp<FORM, true>(g, i, j, k, nullptr, T, BLK_C, y, dA, dC);
    d = (T[o] + y[3]) / dC;
  }
  if ((threadIdx.x & 31) == 0) p[o] += omega * d;
}

}  // namespace stk
