// Fused coarse-level V-cycle: one persistent kernel runs every Uzawa step,
// residual, restriction, coarse solve and prolongation of the levels
// n_l <= fuse_n (V_var schedule R13), separated by software grid
// barriers instead of kernel launches.  On these levels the work per phase is a
// few thousand rows, so launch latency -- not bandwidth -- bounded the
// per-launch kernels (≈ 330 launches per cycle at cfg2).
//
// Rows:
//  * interior rows with an isoviscous star ("regular"): the constant
//    unit stencils st_* (k_assemble_stencils) scaled by mu_k h, h^2, delta h^3/mu_k;
//  * every other row (Gamma_12, Gamma_F, any boundary vertex): an explicit
//    stencil, the 4x4 blocks of K at the 15 Kuhn offsets, assembled once per
//    level by k_assemble_explicit from the element loop ("explicit interface
//    stencils").
// All rows gather the 15-point neighbourhood once (ld.global.cg: data written by
// other CTAs in the previous phase are read from L2, never from a stale L1).
//
// Also: k_gauss_jordan_coop, the coarsest-level inverse (setup) with the same
// grid barrier (the single-CTA version spent ~11 ms in L2 round trips).
#pragma once
#include <cooperative_groups.h>
#include "kernels_generic.cuh"
#include "kernels_tiled.cuh"

namespace stk {

// ---- software grid barrier over the CTA prefix [0, M) -------------------------
// bar[M] is a monotonic 64-bit arrival counter of the prefix [0, M): every CTA
// with index < M calls every barrier with that M in the same order, so the
// counter is a multiple of M between barriers; an arrival adds 1 (release) and
// spins (acquire) until the counter reaches the next multiple of M.  One L2
// atomic per CTA (~1.3 us per barrier on B200, tools/probe_barrier.cu).  M = 1 is
// a CTA barrier.  Co-residency: cooperative launch (cudaLaunchAttributeCooperative).
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, int M) {
  __syncthreads();
  if (M > 1) {
    if (threadIdx.x == 0) {
      unsigned long long* cnt = bar + M;
      unsigned long long old;
      asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
      const unsigned long long target = (old / (unsigned)M + 1) * (unsigned)M;
      while (ld_acquire_u64(cnt) < target) {
      }
    }
    __syncthreads();
  }
}

// one thread per (explicit row, offset q, column field c): row_generic applied to
// the unit vector at (vertex + offset q, field c)
template <int FORM>
__global__ void k_assemble_explicit(DGrid g, const int32_t* __restrict__ rows, int nrows, double* __restrict__ S) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= (int64_t)nrows * NQ * 4) return;
  const int e = (int)(tid / (NQ * 4)), q = (int)((tid / 4) % NQ), c = (int)(tid % 4);
  int i, j, k;
  owned_vertex(g, rows[e], i, j, k);
  FetchUnit fx{i + kq_dx(q), j + kq_dy(q), k + kq_dz(q), c};
  double y[4], dA[3], dC;
  row_generic<FORM>(g, i, j, k, fx, BLK_ALL, y, dA, dC);
  // columns of eliminated neighbour DoFs (Dirichlet / free-slip normal) are 0, as are
  // the rows (row_generic) and inverse diagonals of the row's eliminated components
  const int xi = fx.ui, yj = fx.uj, zk = fx.uk;
  const bool in = xi >= 0 && yj >= 0 && zk >= 0 && xi <= g.n && yj <= g.n && zk <= g.n;
  const bool ecol = c < 3 && (!in || ((elim(g, xi, yj, zk) >> c) & 1u));
#pragma unroll
  for (int r = 0; r < 4; ++r) S[(int64_t)e * EXPL + (r * NQ + q) * 4 + c] = ecol ? 0.0 : y[r];
  if (q == 0 && c == 0) {
    const unsigned em = elim(g, i, j, k);
#pragma unroll
    for (int r = 0; r < 3; ++r) S[(int64_t)e * EXPL + 4 * NQ * 4 + r] = ((em >> r) & 1u) ? 0.0 : 1.0 / dA[r];
    S[(int64_t)e * EXPL + 4 * NQ * 4 + 3] = 1.0 / dC;
  }
}

// rows that need an explicit stencil: Gamma_12 / Gamma_F rows (code >= 0x40: list
// rows and isoviscous traction-face rows).  Interior isoviscous rows use the
// constant stencils; isoviscous Dirichlet-boundary rows (velocity rows 0) the
// interior B stencil on the zero-extended velocity and the truncated C (c_trunc).
__device__ __forceinline__ bool fused_explicit(uint8_t code) { return code >= 0x40; }
__global__ void k_build_explicit(DGrid g, int32_t* __restrict__ slot, int32_t* __restrict__ rows,
                                 unsigned long long* cnt) {
  int i, j, k;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (!owned_vertex(g, t, i, j, k)) return;
  int32_t s = -1;
  if (fused_explicit(g.code[vidx(g, i, j, k)])) {
    s = (int32_t)atomicAdd(cnt, 1ull);
    rows[s] = (int32_t)t;
  }
  slot[vidx(g, i, j, k)] = s;
}

// ---- row kernels of the coarse levels (context-owned vectors) ------------------
// Invariant used throughout: every context-owned level vector is 0
// at Dirichlet velocity DoFs, in the ghost frame and in the spare padding, and the
// halo planes outside the cube are 0 -- every writer below keeps it (Dirichlet
// rows are written as 0, padding is never written).  So the 15-point gather needs
// no masking: out-of-cube and Dirichlet neighbours read as 0.
struct FLevel {
  DGrid g;
  double* x;
  double* b;
  double* r;             // scratch: fields 0..2 velocity ping-pong, field 3 T
  const int32_t* slot;   // padded vertex index -> explicit stencil slot or -1
  const double* S;       // explicit stencils [slot][EXPL]
};

// loads: COH (fused persistent kernel) reads through L2 (ld.global.cg: values
// written by other CTAs in the previous phase); per-phase kernels use the
// read-only path (every kernel launch starts with a clean L1)
template <bool COH>
__device__ __forceinline__ double ldv(const double* p) {
  if (COH) return __ldcg(p);
  return __ldg(p);
}

// 32-bit vertex coordinates of owned linear index t (row levels: < 2^31 vertices)
__device__ __forceinline__ void fvertex(const DGrid& g, int t, int& i, int& j, int& k) {
  const int nx = g.n + 1;
  const int per = nx * nx;
  const int kk = t / per, r = t - kk * per;
  k = g.z0 + kk;
  j = r / nx;
  i = r - j * nx;
}
__device__ __forceinline__ int fidx(const DGrid& g, int i, int j, int k) {
  return (k - g.z0 + 1) * (int)g.py + (j + 1) * (int)g.px + (i + 1);
}

// the 15-point neighbourhood of padded index o (NF = 4: u1,u2,u3,p; NF = 1: p)
template <int NF, bool COH>
__device__ __forceinline__ void gather15(const DGrid& g, int o, const double* U, const double* P,
                                         double nb[NQ][4]) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int oc = o + qoff(g, q);
    if (NF == 4) {
#pragma unroll
      for (int f = 0; f < 3; ++f) nb[q][f] = ldv<COH>(U + f * g.fs + oc);
    } else {
      nb[q][0] = nb[q][1] = nb[q][2] = 0.0;
    }
    nb[q][3] = ldv<COH>(P + oc);
  }
}

// truncated C of an isoviscous boundary vertex (as c_trunc of the tiled kernels):
// sum = sum_e N_e p_e over the 6 axis edges, diag = sum_e N_e
__device__ __forceinline__ void c_trunc_nb(const double nb[NQ][4], int i, int j, int k, int n, double& sum,
                                           double& diag) {
  const int X0 = i >= 1, X1 = i <= n - 1, Y0 = j >= 1, Y1 = j <= n - 1, Z0 = k >= 1, Z1 = k <= n - 1;
  const int wx = 2 * (Y1 & Z1) + (Y0 & Z1) + (Y1 & Z0) + 2 * (Y0 & Z0);
  const int wy = 2 * (X1 & Z1) + (X0 & Z1) + (X1 & Z0) + 2 * (X0 & Z0);
  const int wz = 2 * (X1 & Y1) + (X0 & Y1) + (X1 & Y0) + 2 * (X0 & Y0);
  // q: +x 1, -x 2, +y 3, -y 4, +z 7, -z 8 (absent neighbours are 0)
  sum = wx * (nb[1][3] + nb[2][3]) + wy * (nb[3][3] + nb[4][3]) + wz * (nb[7][3] + nb[8][3]);
  diag = (double)((X0 + X1) * wx + (Y0 + Y1) * wy + (Z0 + Z1) * wz);
}
__device__ __forceinline__ constexpr bool q_axis(int q) { return q == 0 || q == 1 || q == 2 || q == 3 || q == 4 || q == 7 || q == 8; }
__device__ __forceinline__ constexpr int q_o27(int q) { return (kq_dz(q) + 1) * 9 + (kq_dy(q) + 1) * 3 + (kq_dx(q) + 1); }

// rows of K at an owned vertex from the gathered neighbourhood.  ROWS: 1 velocity
// rows (A, B^T), 2 pressure row (B, -C), 3 both; PONLY: the pressure row of C on
// the colour-0 neighbours only (R11).  Velocity rows are 0 at Dirichlet vertices.
// iA, iC: inverse diagonals of A and C (Gauss-Seidel).
template <int FORM, int ROWS, bool PONLY>
__device__ __forceinline__ void row_fused(const FLevel& L, int o, int i, int j, int k, uint8_t code,
                                          const double nb[NQ][4], double y[4], double iA[3], double& iC) {
  const DGrid& g = L.g;
  y[0] = y[1] = y[2] = y[3] = 0.0;
  iA[0] = iA[1] = iA[2] = iC = 0.0;
  const double h = g.h;
  if (code < 0x40) {
    const double mu = mu_of(g, code), imu = imu_of(g, code);
    const double sA = mu * h, sB = h * h, sC = g.delta * h * h * h * imu;
    const bool interior = i > 0 && j > 0 && k > 0 && i < g.n && j < g.n && k < g.n;
    if ((ROWS & 1) && interior) {
      double a[3] = {0, 0, 0}, bt[3] = {0, 0, 0};
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (FORM == FORM_SYM) {
#pragma unroll
            for (int c = 0; c < 3; ++c) a[r] = fma(st_A[FORM][r][c][q_o27(q)], nb[q][c], a[r]);
          } else if (q_axis(q)) {  // 7-point Laplacian (no cross part on isoviscous stars)
            a[r] = fma(st_A[FORM][r][r][q_o27(q)], nb[q][r], a[r]);
          }
          if (q != 0) bt[r] = fma(st_BT[r][q_o27(q)], nb[q][3], bt[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) y[r] = fma(sA, a[r], sB * bt[r]);
      // 1 / (mu h st_A[r][r][centre]), st_A = kst / 6 with integer kst (h = 1/n, n a power of 2)
      const double ia = imu * (double)g.n * 6.0;
      iA[0] = ia * (1.0 / KS<0, FORM, 0, 0, 0, 0, 0>::v);
      iA[1] = ia * (1.0 / KS<0, FORM, 1, 1, 0, 0, 0>::v);
      iA[2] = ia * (1.0 / KS<0, FORM, 2, 2, 0, 0, 0>::v);
    }
    if (ROWS & 2) {
      double bb = 0.0, cc = 0.0;
      if (!PONLY) {
#pragma unroll
        for (int q = 1; q < NQ; ++q)
#pragma unroll
          for (int c = 0; c < 3; ++c) bb = fma(st_B[c][q_o27(q)], nb[q][c], bb);
      }
      if (interior) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q_axis(q) && (!PONLY || q_odd(q))) cc = fma(st_C[q_o27(q)], nb[q][3], cc);
        y[3] = fma(sB, bb, -sC * cc);
        iC = mu * (6.0 / KS<3, 0, 0, 0, 0, 0, 0>::v) / (g.delta * h * h * h);
      } else {
        double sum, diag;
        c_trunc_nb(nb, i, j, k, g.n, sum, diag);  // PONLY: nb[0][3] = 0, axis neighbours are colour 0
        const double cw = sC * (1.0 / 6.0);
        y[3] = fma(sB, bb, -cw * (diag * nb[0][3] - sum));
        iC = 1.0 / (cw * diag);
      }
    }
    return;
  }
  const double* S = L.S + (int64_t)__ldg(L.slot + o) * EXPL;
  if (ROWS & 1) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const double2 s01 = __ldg(reinterpret_cast<const double2*>(S + (r * NQ + q) * 4));
        const double2 s23 = __ldg(reinterpret_cast<const double2*>(S + (r * NQ + q) * 4 + 2));
        acc = fma(s01.x, nb[q][0], acc);
        acc = fma(s01.y, nb[q][1], acc);
        acc = fma(s23.x, nb[q][2], acc);
        acc = fma(s23.y, nb[q][3], acc);
      }
      y[r] = acc;
      iA[r] = __ldg(S + 4 * NQ * 4 + r);
    }
  }
  if (ROWS & 2) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (PONLY && !q_odd(q)) continue;
      const double2 s23 = __ldg(reinterpret_cast<const double2*>(S + (3 * NQ + q) * 4 + 2));
      if (!PONLY) {
        const double2 s01 = __ldg(reinterpret_cast<const double2*>(S + (3 * NQ + q) * 4));
        acc = fma(s01.x, nb[q][0], acc);
        acc = fma(s01.y, nb[q][1], acc);
        acc = fma(s23.x, nb[q][2], acc);
      }
      acc = fma(s23.y, nb[q][3], acc);
    }
    y[3] = acc;
    iC = __ldg(S + 4 * NQ * 4 + 3);
  }
}

// rows t of one phase over `nthr` threads starting at global thread `t0`
#define ROW_LOOP(Lv, t0, nthr) \
  for (int t = (t0), tend = ((Lv).g.n + 1) * ((Lv).g.n + 1) * (Lv).g.nzl; t < tend; t += (nthr))

// one colour pass of the velocity GS (Jacobi within the colour, R12):
// u_out = u_in + (f - A u_in - B^T p) / diag(A) on colour `color`, u_in elsewhere
template <int FORM, bool COH>
__device__ __forceinline__ void f_vel_pass(const FLevel& L, int t0, int nthr, const double* uin, const double* p,
                                           double* uout, int color, int nc) {
  const DGrid& g = L.g;
  ROW_LOOP(L, t0, nthr) {
    int i, j, k;
    fvertex(g, t, i, j, k);
    const int o = fidx(g, i, j, k);
    const unsigned em = elim(g, i, j, k);
    const bool act = ((i + j + k) % nc) == color && em != 7u;
    if (!act) {  // Dirichlet entries of uin are 0 (invariant)
#pragma unroll
      for (int a = 0; a < 3; ++a) uout[a * g.fs + o] = ldv<COH>(uin + a * g.fs + o);
      continue;
    }
    const uint8_t code = __ldg(g.code + o);
    double bv[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) bv[a] = ldv<COH>(L.b + a * g.fs + o);
    double nb[NQ][4], y[4], iA[3], iC;
    gather15<4, COH>(g, o, uin, p, nb);
    row_fused<FORM, 1, false>(L, o, i, j, k, code, nb, y, iA, iC);
#pragma unroll
    for (int a = 0; a < 3; ++a) uout[a * g.fs + o] = fma(bv[a] - y[a], iA[a], nb[0][a]);
  }
}

// pressure pass 1: r_p = B u - C p - g; T = r_p / C_ii (colour 0), r_p (colour 1)
template <int FORM, bool COH>
__device__ __forceinline__ void f_p_pass1(const FLevel& L, int t0, int nthr, const double* x, double* T) {
  const DGrid& g = L.g;
  ROW_LOOP(L, t0, nthr) {
    int i, j, k;
    fvertex(g, t, i, j, k);
    const int o = fidx(g, i, j, k);
    const uint8_t code = __ldg(g.code + o);
    const double gv = ldv<COH>(L.b + 3 * g.fs + o);
    double nb[NQ][4], y[4], iA[3], iC;
    gather15<4, COH>(g, o, x, x + 3 * g.fs, nb);
    row_fused<FORM, 2, false>(L, o, i, j, k, code, nb, y, iA, iC);
    const double r = y[3] - gv;
    T[o] = ((i + j + k) & 1) == 0 ? r * iC : r;
  }
}

// pressure pass 2: delta = T (colour 0), (T - C delta_0) / C_ii (colour 1); p += omega delta
template <int FORM, bool COH>
__device__ __forceinline__ void f_p_pass2(const FLevel& L, int t0, int nthr, const double* T, double* p,
                                          double omega) {
  const DGrid& g = L.g;
  ROW_LOOP(L, t0, nthr) {
    int i, j, k;
    fvertex(g, t, i, j, k);
    const int o = fidx(g, i, j, k);
    const double pv = COH ? __ldcg(p + o) : p[o];
    double d;
    if (((i + j + k) & 1) == 0) {
      d = ldv<COH>(T + o);
    } else {
      const uint8_t code = __ldg(g.code + o);
      double nb[NQ][4], y[4], iA[3], iC;
      gather15<1, COH>(g, o, nullptr, T, nb);
      nb[0][3] = 0.0;  // own value is colour 1: not part of C delta_0
#pragma unroll
      for (int q = 1; q < NQ; ++q)
        if (!q_odd(q)) nb[q][3] = 0.0;
      const double Tv = ldv<COH>(T + o);
      row_fused<FORM, 2, true>(L, o, i, j, k, code, nb, y, iA, iC);
      d = (Tv + y[3]) * iC;
    }
    p[o] = fma(omega, d, pv);
  }
}

// r = b - K x (velocity rows 0 at Dirichlet vertices)
template <int FORM, bool COH>
__device__ __forceinline__ void f_residual(const FLevel& L, int t0, int nthr) {
  const DGrid& g = L.g;
  ROW_LOOP(L, t0, nthr) {
    int i, j, k;
    fvertex(g, t, i, j, k);
    const int o = fidx(g, i, j, k);
    const uint8_t code = __ldg(g.code + o);
    double bv[4];
#pragma unroll
    for (int f = 0; f < 4; ++f) bv[f] = ldv<COH>(L.b + f * g.fs + o);
    double nb[NQ][4], y[4], iA[3], iC;
    gather15<4, COH>(g, o, L.x, L.x + 3 * g.fs, nb);
    row_fused<FORM, 3, false>(L, o, i, j, k, code, nb, y, iA, iC);
    const unsigned em = elim(g, i, j, k);
#pragma unroll
    for (int f = 0; f < 4; ++f) L.r[f * g.fs + o] = ((em >> f) & 1u) ? 0.0 : bv[f] - y[f];
  }
}

// b_c = P^T r_f (as k_restrict) and x_c = 0, over the coarse vertices
template <bool COH>
__device__ __forceinline__ void f_restrict(const FLevel& F, const FLevel& C, int t0, int nthr) {
  const DGrid &gf = F.g, &gc = C.g;
  ROW_LOOP(C, t0, nthr) {
    int I, J, K;
    fvertex(gc, t, I, J, K);
    const unsigned em = elim(gc, I, J, K);
    const int oc = fidx(gc, I, J, K);
    const int of = fidx(gf, 2 * I, 2 * J, 2 * K);
    double v[NQ][4];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int f = 0; f < 4; ++f) v[q][f] = ldv<COH>(F.r + f * gf.fs + of + qoff(gf, q));  // 0 outside (invariant)
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      double e = 0.0;
#pragma unroll
      for (int q = 1; q < NQ; ++q) e += v[q][f];
      C.x[f * gc.fs + oc] = 0.0;
      C.b[f * gc.fs + oc] = ((em >> f) & 1u) ? 0.0 : fma(0.5, e, v[0][f]);
    }
  }
}

// x_f += P x_c (coarse Kuhn-edge midpoints take the mean of the edge ends)
template <bool COH>
__device__ __forceinline__ void f_prolong_add(const FLevel& C, const FLevel& F, int t0, int nthr) {
  const DGrid &gc = C.g, &gf = F.g;
  ROW_LOOP(F, t0, nthr) {
    int i, j, k;
    fvertex(gf, t, i, j, k);
    const int of = fidx(gf, i, j, k);
    const unsigned em = elim(gf, i, j, k);
    const int I = i >> 1, J = j >> 1, K = k >> 1;
    const int di = i & 1, dj = j & 1, dk = k & 1;
    const int o0 = fidx(gc, I, J, K);
    const bool mid = di | dj | dk;
    const int o1 = mid ? fidx(gc, I + di, J + dj, K + dk) : o0;
    double xf[4], c0[4], c1[4];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      xf[f] = COH ? __ldcg(F.x + f * gf.fs + of) : F.x[f * gf.fs + of];
      c0[f] = ldv<COH>(C.x + f * gc.fs + o0);
      c1[f] = ldv<COH>(C.x + f * gc.fs + o1);
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double v = mid ? 0.5 * (c0[f] + c1[f]) : c0[f];
      F.x[f * gf.fs + of] = ((em >> f) & 1u) ? 0.0 : xf[f] + v;
    }
  }
}

// x_F = G b_F on the coarsest level: one warp per coarse DoF row; x is 0 elsewhere
// (f_restrict zeroed it).  w0/nw: this thread's first warp and the warp count.
template <bool COH>
__device__ __forceinline__ void f_coarse(const FLevel& L, const int32_t* dofs, const double* G, int N, int ld, int w0,
                                         int nw) {
  const DGrid& g = L.g;
  const int lane = threadIdx.x & 31;
  auto at = [&](int32_t d) {
    const int f = (d >> 28) & 0xF, k = (d >> 18) & 0x3FF, j = (d >> 9) & 0x1FF, i = d & 0x1FF;
    return f * (int)g.fs + fidx(g, i, j, k);
  };
  for (int r = w0; r < N; r += nw) {
    double s = 0.0;
    for (int c = lane; c < N; c += 32) s = fma(__ldg(G + (int64_t)r * ld + c), ldv<COH>(L.b + at(__ldg(dofs + c))), s);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) L.x[at(__ldg(dofs + r))] = s;
  }
}

template <bool COH>
__device__ __forceinline__ void f_zero(const FLevel& L, int t0, int nthr) {
  ROW_LOOP(L, t0, nthr) {
    int i, j, k;
    fvertex(L.g, t, i, j, k);
    const int o = fidx(L.g, i, j, k);
#pragma unroll
    for (int f = 0; f < 4; ++f) L.x[f * L.g.fs + o] = 0.0;
  }
}

// ---- per-phase kernels (one launch per phase; captured into the coarse graph) ----
constexpr int ROW_NT = 128;
enum { FPH_ZERO = 0, FPH_VEL, FPH_P1, FPH_P2, FPH_RES, FPH_RESTRICT, FPH_PROLONG, FPH_COARSE };
template <int FORM, int OP>
__global__ void __launch_bounds__(ROW_NT) k_row(const __grid_constant__ FLevel L, const __grid_constant__ FLevel L2,
                                                const double* uin, double* uout, int color, int nc, double omega) {
  const int t0 = blockIdx.x * ROW_NT + threadIdx.x, nthr = gridDim.x * ROW_NT;
  if (OP == FPH_VEL) f_vel_pass<FORM, false>(L, t0, nthr, uin, L.x + 3 * L.g.fs, uout, color, nc);
  if (OP == FPH_P1) f_p_pass1<FORM, false>(L, t0, nthr, L.x, L.r + 3 * L.g.fs);
  if (OP == FPH_P2) f_p_pass2<FORM, false>(L, t0, nthr, L.r + 3 * L.g.fs, L.x + 3 * L.g.fs, omega);
  if (OP == FPH_RES) f_residual<FORM, false>(L, t0, nthr);
  if (OP == FPH_RESTRICT) f_restrict<false>(L, L2, t0, nthr);   // L fine, L2 coarse
  if (OP == FPH_PROLONG) f_prolong_add<false>(L2, L, t0, nthr); // L fine, L2 coarse
}
__global__ void __launch_bounds__(256) k_coarse_warp(const __grid_constant__ FLevel L, const int32_t* dofs,
                                                     const double* G, int N, int ld) {
  f_coarse<false>(L, dofs, G, N, ld, (blockIdx.x * 256 + threadIdx.x) >> 5, gridDim.x * 8);
}

// ---- lane-split row kernels: LPR lanes per row ---------------------------------
// On the small levels a phase is a few thousand rows, so its time is the latency of
// ONE row, not bandwidth: one thread per row runs ~700 dependent instructions
// (ncu: ~19 cycles each at one warp per SMSP).  Here lane q of a row's LPR-lane
// group takes the Kuhn offsets q, q + LPR, ...: it loads its neighbours' 4 fields
// (and, on explicit rows, its 16 stencil entries), forms its part of the 4 row
// outputs, and the group sums them with LPR-segment xor shuffles; lane 0 finishes.

// unit stencils of the interior vertex per Kuhn offset q (compile time, from kst)
struct KTab {
  double A[3][NQ][3][3];  // [form][q][a][b]   6 A / 6
  double BT[NQ][3];       // velocity row a     24 B^T / 24
  double B[NQ][3];        // velocity column b  24 B / 24
  double C[NQ];           //                    6 C / 6
};
constexpr KTab make_ktab() {
  KTab t{};
  for (int q = 0; q < NQ; ++q) {
    const int dx = kq_dx(q), dy = kq_dy(q), dz = kq_dz(q);
    for (int f = 0; f < 3; ++f)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) t.A[f][q][a][b] = kst(0, f, a, b, dx, dy, dz) / 6.0;
    for (int a = 0; a < 3; ++a) {
      t.BT[q][a] = kst(1, 0, a, 0, dx, dy, dz) / 24.0;
      t.B[q][a] = kst(2, 0, 0, a, dx, dy, dz) / 24.0;
    }
    t.C[q] = kst(3, 0, 0, 0, dx, dy, dz) / 6.0;
  }
  return t;
}
__device__ const KTab g_ktab = make_ktab();

template <int LPR>
__device__ __forceinline__ double seg_sum(double v) {
#pragma unroll
  for (int off = LPR / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// partial rows of K from this lane's offsets.  ROWS: 1 velocity rows, 2 pressure
// row, 3 both; PONLY: C on colour-0 neighbours only (R11).  Regular rows (code <
// 0x40) use g_ktab scaled by mu h, h^2, delta h^3/mu; isoviscous boundary rows
// the interior B on the zero-extended velocity and the truncated C (c_trunc).
// Returns the group sums in y[0..3] on every lane of the group.
template <int FORM, int ROWS, bool PONLY, int LPR>
__device__ __forceinline__ void row_lanes(const FLevel& L, const MuTab& M, int o, int i, int j, int k, uint8_t code,
                                          int slot, int sub, const double* U, const double* P, double y[4]) {
  const DGrid& g = L.g;
  double py[4] = {0.0, 0.0, 0.0, 0.0};
  const bool expl = code >= 0x40;
  const double* S = expl ? L.S + (int64_t)slot * EXPL : nullptr;
  const double h = g.h;
  const bool interior = i > 0 && j > 0 && k > 0 && i < g.n && j < g.n && k < g.n;
  double sA = 0.0, sB = h * h, sC = 0.0, cw = 0.0;
  int wq[3] = {0, 0, 0};
  double diag = 0.0;
  if (!expl) {
    sA = M.mu[code] * h;
    sC = g.delta * h * h * h * M.imu[code];
    if (!interior && (ROWS & 2)) {
      const int X0 = i >= 1, X1 = i <= g.n - 1, Y0 = j >= 1, Y1 = j <= g.n - 1, Z0 = k >= 1, Z1 = k <= g.n - 1;
      wq[0] = 2 * (Y1 & Z1) + (Y0 & Z1) + (Y1 & Z0) + 2 * (Y0 & Z0);
      wq[1] = 2 * (X1 & Z1) + (X0 & Z1) + (X1 & Z0) + 2 * (X0 & Z0);
      wq[2] = 2 * (X1 & Y1) + (X0 & Y1) + (X1 & Y0) + 2 * (X0 & Y0);
      diag = (double)((X0 + X1) * wq[0] + (Y0 + Y1) * wq[1] + (Z0 + Z1) * wq[2]);
      cw = sC * (1.0 / 6.0);
    }
  }
#pragma unroll
  for (int qq = 0; qq < (NQ + LPR - 1) / LPR; ++qq) {
    const int q = sub + qq * LPR;
    if (q >= NQ) break;
    const int oc = o + qoff(g, q);
    const int dsum = kq_dx(q) + kq_dy(q) + kq_dz(q);
    double u[3] = {0.0, 0.0, 0.0}, pv;
    if (!PONLY) {
#pragma unroll
      for (int c = 0; c < 3; ++c) u[c] = __ldg(U + c * g.fs + oc);
    }
    pv = __ldg(P + oc);
    if (PONLY && !(dsum & 1)) pv = 0.0;  // colour-1 own value and even offsets: not colour 0
    if (expl) {
      if (ROWS & 1) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double2 s01 = __ldg(reinterpret_cast<const double2*>(S + (r * NQ + q) * 4));
          const double2 s23 = __ldg(reinterpret_cast<const double2*>(S + (r * NQ + q) * 4 + 2));
          py[r] = fma(s01.x, u[0], fma(s01.y, u[1], fma(s23.x, u[2], s23.y * pv)));
        }
      }
      if (ROWS & 2) {
        const double2 s23 = __ldg(reinterpret_cast<const double2*>(S + (3 * NQ + q) * 4 + 2));
        double acc = s23.y * pv;
        if (!PONLY) {
          const double2 s01 = __ldg(reinterpret_cast<const double2*>(S + (3 * NQ + q) * 4));
          acc = fma(s01.x, u[0], fma(s01.y, u[1], fma(s23.x, u[2], acc)));
        }
        py[3] += acc;
      }
    } else {
      if ((ROWS & 1) && interior) {
        const double* A = &g_ktab.A[FORM][q][0][0];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          double a;
          if (FORM == FORM_SYM) a = fma(__ldg(A + r * 3 + 0), u[0], fma(__ldg(A + r * 3 + 1), u[1], __ldg(A + r * 3 + 2) * u[2]));
          else a = __ldg(A + r * 3 + r) * u[r];
          py[r] += fma(sA, a, sB * __ldg(&g_ktab.BT[q][r]) * pv);
        }
      }
      if (ROWS & 2) {
        double bb = 0.0;
        if (!PONLY) bb = fma(__ldg(&g_ktab.B[q][0]), u[0], fma(__ldg(&g_ktab.B[q][1]), u[1], __ldg(&g_ktab.B[q][2]) * u[2]));
        double cc;
        if (interior) {
          cc = -sC * __ldg(&g_ktab.C[q]) * pv;
        } else {
          // truncated C: -cw (diag p_v - sum_e N_e p_e); q: +-x 1,2; +-y 3,4; +-z 7,8
          const int ax = (q == 1 || q == 2) ? 0 : (q == 3 || q == 4) ? 1 : (q == 7 || q == 8) ? 2 : -1;
          cc = q == 0 ? -cw * diag * pv : ax >= 0 ? cw * wq[ax] * pv : 0.0;
        }
        py[3] += fma(sB, bb, cc);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if ((r < 3 && (ROWS & 1)) || (r == 3 && (ROWS & 2))) py[r] = seg_sum<LPR>(py[r]);
#pragma unroll
  for (int r = 0; r < 4; ++r) y[r] = py[r];
  if (!expl && !interior) y[0] = y[1] = y[2] = 0.0;  // Dirichlet velocity rows
}
// inverse diagonals of a row (lane 0 of the group)
template <int FORM>
__device__ __forceinline__ void row_inv_diag(const FLevel& L, const MuTab& M, int o, int i, int j, int k, uint8_t code,
                                             int slot, double iA[3], double& iC) {
  const DGrid& g = L.g;
  if (code >= 0x40) {
    const double* S = L.S + (int64_t)slot * EXPL + 4 * NQ * 4;
    iA[0] = __ldg(S);
    iA[1] = __ldg(S + 1);
    iA[2] = __ldg(S + 2);
    iC = __ldg(S + 3);
    return;
  }
  const double h = g.h, mu = M.mu[code];
  const double ia = M.imu[code] * (double)g.n * 6.0;
  iA[0] = ia * (1.0 / KS<0, FORM, 0, 0, 0, 0, 0>::v);
  iA[1] = ia * (1.0 / KS<0, FORM, 1, 1, 0, 0, 0>::v);
  iA[2] = ia * (1.0 / KS<0, FORM, 2, 2, 0, 0, 0>::v);
  const bool interior = i > 0 && j > 0 && k > 0 && i < g.n && j < g.n && k < g.n;
  if (interior) {
    iC = mu * (6.0 / KS<3, 0, 0, 0, 0, 0, 0>::v) / (g.delta * h * h * h);
  } else {
    const int X0 = i >= 1, X1 = i <= g.n - 1, Y0 = j >= 1, Y1 = j <= g.n - 1, Z0 = k >= 1, Z1 = k <= g.n - 1;
    const int wx = 2 * (Y1 & Z1) + (Y0 & Z1) + (Y1 & Z0) + 2 * (Y0 & Z0);
    const int wy = 2 * (X1 & Z1) + (X0 & Z1) + (X1 & Z0) + 2 * (X0 & Z0);
    const int wz = 2 * (X1 & Y1) + (X0 & Y1) + (X1 & Y0) + 2 * (X0 & Y0);
    const double diag = (double)((X0 + X1) * wx + (Y0 + Y1) * wy + (Z0 + Z1) * wz);
    iC = 6.0 * mu / (g.delta * h * h * h * diag);
  }
}

// one phase over LPR-lane row groups; every lane of a group runs the same control
// flow up to the shuffles (the row index is uniform within the group)
template <int FORM, int OP, int LPR>
__global__ void __launch_bounds__(ROW_NT) k_rowl(const __grid_constant__ FLevel L, const __grid_constant__ FLevel L2,
                                                 const double* uin, double* uout, int color, int nc, double omega,
                                                 const __grid_constant__ MuTab M) {
  const int gt = blockIdx.x * ROW_NT + threadIdx.x;
  const int sub = gt & (LPR - 1);
  const DGrid& g = L.g;
  const int nx = g.n + 1;
  const int rows = (OP == FPH_RESTRICT ? (L2.g.n + 1) * (L2.g.n + 1) * L2.g.nzl : nx * nx * g.nzl);
  const int t = gt / LPR;
  if (t >= rows) return;  // whole groups retire together (rows are group-uniform)
  if (OP == FPH_RESTRICT) {  // b_c = R r_f, x_c = 0 (L fine, L2 coarse)
    const DGrid& gc = L2.g;
    int I, J, K;
    fvertex(gc, t, I, J, K);
    const int oc = fidx(gc, I, J, K);
    const int of = fidx(g, 2 * I, 2 * J, 2 * K);
    double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int qq = 0; qq < (NQ + LPR - 1) / LPR; ++qq) {
      const int q = sub + qq * LPR;
      if (q >= NQ) break;
      const double w = q == 0 ? 1.0 : 0.5;
#pragma unroll
      for (int f = 0; f < 4; ++f) v[f] = fma(w, __ldg(L.r + f * g.fs + of + qoff(g, q)), v[f]);  // 0 outside
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) v[f] = seg_sum<LPR>(v[f]);
    if (sub < 4) {
      const unsigned em = elim(gc, I, J, K);
      L2.x[sub * gc.fs + oc] = 0.0;
      const double vv = sub == 0 ? v[0] : sub == 1 ? v[1] : sub == 2 ? v[2] : v[3];
      L2.b[sub * gc.fs + oc] = ((em >> sub) & 1u) ? 0.0 : vv;
    }
    return;
  }
  int i, j, k;
  fvertex(g, t, i, j, k);
  const int o = fidx(g, i, j, k);
  if (OP == FPH_VEL) {
    const unsigned em = elim(g, i, j, k);
    const bool act = ((i + j + k) % nc) == color && em != 7u;
    if (!act) {  // Dirichlet entries of uin are 0 (invariant)
      if (sub < 3) uout[sub * g.fs + o] = __ldg(uin + sub * g.fs + o);
      return;
    }
    const uint8_t code = __ldg(g.code + o);
    const int slot = __ldg(L.slot + o);  // independent of code: one round trip for both
    const int c3 = sub < 3 ? sub : 0;
    const double bown = __ldg(L.b + c3 * g.fs + o), uown = __ldg(uin + c3 * g.fs + o);  // issued early
    double y[4];
    row_lanes<FORM, 1, false, LPR>(L, M, o, i, j, k, code, slot, sub, uin, L.x + 3 * g.fs, y);
    if (sub < 3) {
      double iA[3], iC;
      row_inv_diag<FORM>(L, M, o, i, j, k, code, slot, iA, iC);
      const double yv = sub == 0 ? y[0] : sub == 1 ? y[1] : y[2];
      const double ia = sub == 0 ? iA[0] : sub == 1 ? iA[1] : iA[2];
      uout[sub * g.fs + o] = fma(bown - yv, ia, uown);
    }
  } else if (OP == FPH_P1) {  // T = (B u - C p - g) / C_ii on colour 0, unscaled on colour 1
    const uint8_t code = __ldg(g.code + o);
    const int slot = __ldg(L.slot + o);
    double y[4];
    row_lanes<FORM, 2, false, LPR>(L, M, o, i, j, k, code, slot, sub, L.x, L.x + 3 * g.fs, y);
    if (sub == 0) {
      const double r = y[3] - __ldg(L.b + 3 * g.fs + o);
      double iA[3], iC = 1.0;
      if (((i + j + k) & 1) == 0) row_inv_diag<FORM>(L, M, o, i, j, k, code, slot, iA, iC);
      L.r[3 * g.fs + o] = ((i + j + k) & 1) == 0 ? r * iC : r;
    }
  } else if (OP == FPH_P2) {  // p += omega delta
    double* p = L.x + 3 * g.fs;
    const double* T = L.r + 3 * g.fs;
    if (((i + j + k) & 1) == 0) {
      if (sub == 0) p[o] = fma(omega, __ldg(T + o), p[o]);
      return;
    }
    const uint8_t code = __ldg(g.code + o);
    const int slot = __ldg(L.slot + o);
    double y[4];
    row_lanes<FORM, 2, true, LPR>(L, M, o, i, j, k, code, slot, sub, nullptr, T, y);
    if (sub == 0) {
      double iA[3], iC;
      row_inv_diag<FORM>(L, M, o, i, j, k, code, slot, iA, iC);
      p[o] = fma(omega, (__ldg(T + o) + y[3]) * iC, p[o]);
    }
  } else if (OP == FPH_RES) {  // r = b - K x
    const uint8_t code = __ldg(g.code + o);
    const int slot = __ldg(L.slot + o);
    double y[4];
    row_lanes<FORM, 3, false, LPR>(L, M, o, i, j, k, code, slot, sub, L.x, L.x + 3 * g.fs, y);
    if (sub < 4) {
      const unsigned em = elim(g, i, j, k);
      const double yv = sub == 0 ? y[0] : sub == 1 ? y[1] : sub == 2 ? y[2] : y[3];
      L.r[sub * g.fs + o] = ((em >> sub) & 1u) ? 0.0 : __ldg(L.b + sub * g.fs + o) - yv;
    }
  } else if (OP == FPH_PROLONG) {  // x_f += P x_c (L fine, L2 coarse)
    if (sub < 4) {
      const DGrid& gc = L2.g;
      const int f = sub;
      const unsigned em = elim(g, i, j, k);
      const int I = i >> 1, J = j >> 1, K = k >> 1;
      const int di = i & 1, dj = j & 1, dk = k & 1;
      const int o0 = fidx(gc, I, J, K);
      const bool mid = di | dj | dk;
      const int o1 = mid ? fidx(gc, I + di, J + dj, K + dk) : o0;
      const double c0 = __ldg(L2.x + f * gc.fs + o0), c1 = __ldg(L2.x + f * gc.fs + o1);
      const double v = mid ? 0.5 * (c0 + c1) : c0;
      L.x[f * g.fs + o] = ((em >> f) & 1u) ? 0.0 : L.x[f * g.fs + o] + v;
    }
  }
}

// ---- fused persistent V-cycle (optional, stk_set_fuse_n) ------------------------
constexpr int FMAX = 8;
constexpr int FCL = 16;  // CTAs of the fused V-cycle's thread-block cluster (non-portable size)
// one phase of the fused V-cycle (built on the host, read from shared memory)
struct FPhase {
  uint8_t op, lev, color, flip;  // flip (FPH_VEL): input in the scratch vector, output in x
  int16_t m;                      // participating CTAs
  int16_t barM;                   // barrier after the phase over CTAs [0, barM) (0: none)
};
constexpr int FPH_MAX = 1024;
struct FusedArgs {
  FLevel L[FMAX];
  int nl;                // levels in the fused part (the last is the coarsest)
  int nph;
  const FPhase* prog;    // device array [nph]
  int ncolors;
  double omega;
  // coarsest level dense solve x_F = G b_F
  const int32_t* cdofs;
  const double* cG;
  int cN, cld;
  unsigned long long* bar;
  unsigned long long* trace;  // debug (STK_FUSED_TRACE): globaltimer after every phase, CTA 0
  int cluster;                // 1: the grid is one thread-block cluster, phases end at a cluster barrier
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// The V-cycle of the fused levels on L[0].b from x = 0 (the caller restricted into
// L[0].b): the phase program (zero; per level nu Uzawa steps = 2 nc velocity
// passes + 2 pressure passes, residual, restriction; coarse solve; per level
// prolongation + nu Uzawa steps) is read into shared memory once.
template <int FORM>
__global__ void __launch_bounds__(256, 1) k_mg_fused(const __grid_constant__ FusedArgs A) {
  __shared__ FPhase prog[FPH_MAX];
  __shared__ FLevel lev[FMAX];
  for (int q = threadIdx.x; q < A.nph; q += blockDim.x) prog[q] = A.prog[q];
  if (threadIdx.x < A.nl) lev[threadIdx.x] = A.L[threadIdx.x];
  __syncthreads();
  const bool tr = A.trace && blockIdx.x == 0 && threadIdx.x == 0;
  if (tr) A.trace[FPH_MAX] = globaltimer();
  for (int ph = 0; ph < A.nph; ++ph) {
    const FPhase P = prog[ph];
    if ((int)blockIdx.x < P.m) {
      const FLevel& L = lev[P.lev];
      const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nthr = P.m * blockDim.x;
      switch (P.op) {
        case FPH_ZERO: f_zero<true>(L, t0, nthr); break;
        case FPH_VEL: {
          double* tmp = L.r;
          f_vel_pass<FORM, true>(L, t0, nthr, P.flip ? tmp : L.x, L.x + 3 * L.g.fs, P.flip ? L.x : tmp, P.color,
                                 A.ncolors);
          break;
        }
        case FPH_P1: f_p_pass1<FORM, true>(L, t0, nthr, L.x, L.r + 3 * L.g.fs); break;
        case FPH_P2: f_p_pass2<FORM, true>(L, t0, nthr, L.r + 3 * L.g.fs, L.x + 3 * L.g.fs, A.omega); break;
        case FPH_RES: f_residual<FORM, true>(L, t0, nthr); break;
        case FPH_RESTRICT: f_restrict<true>(L, lev[P.lev + 1], t0, nthr); break;
        case FPH_PROLONG: f_prolong_add<true>(lev[P.lev + 1], L, t0, nthr); break;
        default: f_coarse<true>(L, A.cdofs, A.cG, A.cN, A.cld, t0 >> 5, nthr >> 5); break;
      }
    }
    if (A.cluster) {
      cooperative_groups::this_cluster().sync();  // hardware barrier; release/acquire at cluster scope
    } else if (P.barM > 0 && (int)blockIdx.x < P.barM) {
      grid_barrier(A.bar, P.barM);
    }
    if (tr) A.trace[ph] = globaltimer();
  }
}

// ---- coarsest-level inverse on one thread-block cluster (distributed shared memory) ----
// In-place Gauss-Jordan with partial pivoting: CTA r of the GJC-CTA cluster holds rows
// [r R, (r+1) R) of the N x N matrix in its shared memory.  Per column k: every CTA
// offers its best pivot candidate (|A[i][k]|, i >= k) to CTA 0 -> cluster barrier ->
// every CTA picks the pivot row p (ties -> lowest index), reads row p remotely and
// forms the scaled pivot row (A[k][k] -> 1/piv, others / piv) in its own buffer; the
// owner of p keeps a copy of row k -> cluster barrier -> the owners write the swapped
// rows, every CTA eliminates its other rows with its pivot-row copy.  Two cluster
// barriers per column (the grid version needed two grid barriers plus a one-CTA
// pivot phase).  Column interchanges are undone at the end (Numerical-Recipes order).
constexpr int GJC = 8, GJC_NT = 256;
inline size_t gj_cluster_smem(int N) {
  const int R = (N + GJC - 1) / GJC;
  return sizeof(double) * ((size_t)R * N + 2 * (size_t)N + GJC) + sizeof(int) * (GJC + N + 8);
}
__global__ void __cluster_dims__(GJC, 1, 1) __launch_bounds__(GJC_NT)
    k_gauss_jordan_cluster(const double* __restrict__ K, double* __restrict__ G, int N, int* status) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int R = (N + GJC - 1) / GJC;
  const int r0 = rank * R, r1 = min(N, r0 + R);
  extern __shared__ double gsm[];
  double* A = gsm;                    // [R][N] own rows
  double* prow = A + (size_t)R * N;   // scaled pivot row (private copy)
  double* keep = prow + N;            // old row k (owner of row p only)
  double* cval = keep + N;            // [GJC] candidates (CTA 0's copy is read)
  int* cidx = reinterpret_cast<int*>(cval + GJC);
  int* perm = cidx + GJC;             // [N] pivot rows
  __shared__ double wv[GJC_NT / 32];
  __shared__ int wi[GJC_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < (r1 - r0) * N; e += GJC_NT) A[e] = K[(size_t)(r0 + e / N) * N + e % N];
  __syncthreads();
  for (int k = 0; k < N; ++k) {
    // local pivot candidate among own rows i >= k
    double bv = -1.0;
    int bi = N;
    for (int i = max(r0, k) + tid; i < r1; i += GJC_NT) {
      const double v = fabs(A[(size_t)(i - r0) * N + k]);
      if (v > bv) { bv = v; bi = i; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { wv[wid] = bv; wi[wid] = bi; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < GJC_NT / 32; ++w)
        if (wv[w] > bv || (wv[w] == bv && wi[w] < bi)) { bv = wv[w]; bi = wi[w]; }
      double* rv = cl.map_shared_rank(cval, 0);
      int* ri = cl.map_shared_rank(cidx, 0);
      rv[rank] = bv;
      ri[rank] = bi;
    }
    cl.sync();
    // global pivot: lanes 0..GJC-1 of warp 0 read CTA 0's candidates in parallel
    __shared__ int psh;
    if (wid == 0) {
      const double* rv = cl.map_shared_rank(cval, 0);
      const int* ri = cl.map_shared_rank(cidx, 0);
      double gv = lane < GJC ? rv[lane] : -1.0;
      int gp = lane < GJC ? ri[lane] : N;
#pragma unroll
      for (int off = GJC / 2; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, gv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, gp, off);
        if (ov > gv || (ov == gv && oi < gp)) { gv = ov; gp = oi; }
      }
      if (lane == 0) {
        psh = gp;
        if (rank == 0 && !(gv > 0.0)) *status = 1;
      }
    }
    __syncthreads();
    const int p = psh;
    const int op = p / R, ok = k / R;
    const double* rowp = cl.map_shared_rank(A, op) + (size_t)(p - op * R) * N;
    const double piv = rowp[k];
    const double ipiv = 1.0 / piv;
    for (int j = tid; j < N; j += GJC_NT) prow[j] = j == k ? ipiv : rowp[j] * ipiv;
    if (rank == op && p != k) {
      const double* rowk = cl.map_shared_rank(A, ok) + (size_t)(k - ok * R) * N;
      for (int j = tid; j < N; j += GJC_NT) keep[j] = rowk[j];
    }
    if (tid == 0) perm[k] = p;
    cl.sync();
    if (rank == ok)
      for (int j = tid; j < N; j += GJC_NT) A[(size_t)(k - r0) * N + j] = prow[j];
    if (rank == op && p != k)
      for (int j = tid; j < N; j += GJC_NT) A[(size_t)(p - r0) * N + j] = keep[j];
    __syncthreads();
    // eliminate column k from the own rows i != k: A[i][k] -> -f / piv, A[i][j] -= f prow[j]
    const int nr = r1 - r0;
    for (int w = wid; w < nr; w += GJC_NT / 32) {
      const int i = r0 + w;
      if (i == k) continue;
      double* ai = A + (size_t)w * N;
      const double f = ai[k];
      if (f == 0.0) continue;
      for (int j = lane; j < N; j += 32) ai[j] = j == k ? -f * prow[k] : fma(-f, prow[j], ai[j]);
    }
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, in reverse order
  for (int k = N - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p == k) continue;
    for (int w = tid; w < r1 - r0; w += GJC_NT) {
      double* ai = A + (size_t)w * N;
      const double t = ai[k];
      ai[k] = ai[p];
      ai[p] = t;
    }
    __syncthreads();
  }
  for (int e = tid; e < (r1 - r0) * N; e += GJC_NT) G[(size_t)(r0 + e / N) * N + e % N] = A[e];
  cl.sync();  // no CTA leaves while its shared memory may still be read remotely
}

// ---- coarsest-level inverse: Gauss-Jordan with partial pivoting, grid-parallel ----
// Per column c: CTA 0 picks the pivot (largest |A[r][c]|, r >= c, ties -> lowest r),
// swaps rows c and p of A and Inv, scales row c by 1/A[c][c] and saves the column
// factors fac[r] = A[r][c]; after a barrier every CTA eliminates its share of the
// other rows; after a second barrier the next column starts.
__global__ void __launch_bounds__(256, 1) k_gauss_jordan_coop(double* __restrict__ A, double* __restrict__ Inv,
                                                              double* __restrict__ fac, int N, int* status,
                                                              unsigned long long* bar) {
  const int G = gridDim.x;
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)G * blockDim.x;
  for (int64_t e = gt; e < (int64_t)N * N; e += gs) Inv[e] = (e / N == e % N) ? 1.0 : 0.0;
  __shared__ double redv[256];
  __shared__ int redi[256];
  grid_barrier(bar, G);
  for (int c = 0; c < N; ++c) {
    if (blockIdx.x == 0) {
      double best = -1.0;
      int bi = c;
      for (int r = c + threadIdx.x; r < N; r += blockDim.x) {
        const double v = fabs(__ldcg(A + (int64_t)r * N + c));
        if (v > best) { best = v; bi = r; }
      }
      redv[threadIdx.x] = best;
      redi[threadIdx.x] = bi;
      __syncthreads();
      for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s && (redv[threadIdx.x + s] > redv[threadIdx.x] ||
                                (redv[threadIdx.x + s] == redv[threadIdx.x] && redi[threadIdx.x + s] < redi[threadIdx.x]))) {
          redv[threadIdx.x] = redv[threadIdx.x + s];
          redi[threadIdx.x] = redi[threadIdx.x + s];
        }
        __syncthreads();
      }
      const int p = redi[0];
      if (threadIdx.x == 0 && !(redv[0] > 0.0)) *status = 1;
      const double d = __ldcg(A + (int64_t)p * N + c);
      for (int q = threadIdx.x; q < N; q += blockDim.x) {
        const double ac = __ldcg(A + (int64_t)c * N + q), ap = __ldcg(A + (int64_t)p * N + q);
        const double ic = __ldcg(Inv + (int64_t)c * N + q), ip = __ldcg(Inv + (int64_t)p * N + q);
        A[(int64_t)c * N + q] = ap / d;
        Inv[(int64_t)c * N + q] = ip / d;
        if (p != c) {
          A[(int64_t)p * N + q] = ac;
          Inv[(int64_t)p * N + q] = ic;
        }
      }
      __syncthreads();
      for (int r = threadIdx.x; r < N; r += blockDim.x)
        fac[r] = r == c ? 0.0 : __ldcg(A + (int64_t)r * N + c);
    }
    grid_barrier(bar, G);
    for (int64_t e = gt; e < (int64_t)N * N; e += gs) {
      const int r = (int)(e / N), q = (int)(e % N);
      if (r == c) continue;
      const double f = __ldcg(fac + r);
      if (f == 0.0) continue;
      A[e] = __ldcg(A + e) - f * __ldcg(A + (int64_t)c * N + q);
      Inv[e] = __ldcg(Inv + e) - f * __ldcg(Inv + (int64_t)c * N + q);
    }
    grid_barrier(bar, G);
  }
}

}  // namespace stk
