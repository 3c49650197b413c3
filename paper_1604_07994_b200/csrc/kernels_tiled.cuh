// Tiled constant-stencil kernels for levels with n >= 64 (the hot path).
//
// Design:
//  * One launch = two CTA roles.  The first `list_blocks` CTAs evaluate the
//    rows of the compact list of irregular vertices (interface Gamma_12, the
//    traction boundary Gamma_F, vertices touching both kinds of faces) by the
//    element loop row_generic, one row per thread, reading the input vector
//    from global memory (L2).  The remaining CTAs stream the grid.  The two
//    write disjoint rows, so they need no synchronisation and the hardware
//    back-fills stream CTAs as soon as the list CTAs retire.
//  * A stream CTA owns a TX x TY column tile (i in [i0, i0+TX), j in
//    [j0, j0+TY), i0+TX <= n) and a chunk of z-planes.  Each plane of the input
//    fields, with a 1-vertex xy halo, is staged in shared memory by TMA boxes
//    (cp.async.bulk.tensor.4d + mbarrier complete_tx), PREF planes ahead, in a
//    ring of PREF+2 slots.  One __syncthreads per plane.
//  * Plane-streaming accumulation: when plane P lands, every thread reads the
//    7 in-plane points of its column once and adds their contributions to the
//    rows of outputs P-1, P, P+1 of its column (the 15-point Kuhn stencil
//    spans three planes).  HBM traffic: one read of x, one write of y.
//  * Regular rows (isoviscous star of class k) use the constant
//    unit stencils assembled once by k_assemble_stencils, scaled by mu_k h
//    (A), h^2 (B, B^T) and delta h^3 / mu_k (C).
//  * Dirichlet boundary rows with an isoviscous star stay in the stream: their
//    velocity rows are 0 and the pressure row is B u - C_trunc p, where B u is
//    the full interior B stencil applied to the zero-extended velocity (the
//    tets outside the cube only touch Dirichlet vertices, so they add 0) and
//    C_trunc has the edge weights (delta h^3 / 6 mu) N_e, N_e = number of tets
//    inside the cube around edge e.  The velocity tensor map
//    starts/ends one vertex inside every Dirichlet face, so TMA's out-of-bounds
//    zero fill applies the Dirichlet condition to the staged planes for free.
//  * The face column i = n and the face row j = n are the right/top halo of the
//    last tiles; their (Dirichlet) rows are finished by one lane / one warp.
#pragma once
#include <cuda.h>

#include <cstdlib>

#include "stk_common.cuh"

namespace stk {

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int HX = TX + 2, HY = TY + 2, PLANE = HX * HY;
// shared-memory stride of one staged field plane: 128-byte aligned TMA destinations
constexpr int FST = ((PLANE + 15) / 16) * 16;
constexpr int PREF = 3, RING = PREF + 2;

// unit stencils (h = 1, mu = 1, delta = 1) of an interior vertex, offset index
// o = (dz+1)*9 + (dy+1)*3 + (dx+1):  row (centre, a) / centre pressure row
__constant__ double st_A[3][3][3][27];  // [form][a][b][o]
__constant__ double st_BT[3][27];       // velocity row a, pressure column
__constant__ double st_B[3][27];        // pressure row, velocity column b
__constant__ double st_C[27];

enum { OP_APPLY = 0, OP_RESID = 1, OP_VEL = 2, OP_P1 = 3, OP_P2 = 4 };

// one thread: unit stencils of the interior vertex by summing the element
// matrices of its 24 incident tetrahedra (the "constant subdomain stencils")
__global__ void k_assemble_stencils(double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double A[3][3][3][27] = {}, BT[3][27] = {}, B[3][27] = {}, C[27] = {};
  const double vol = 1.0 / 6.0;
  for (int dz = -1; dz <= 0; ++dz)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dx = -1; dx <= 0; ++dx) {
        const int corner = (-dx) | ((-dy) << 1) | ((-dz) << 2);
        for (int t = 0; t < 6; ++t) {
          const int m = c_corner_m[corner][t];
          if (m < 0) continue;
          const int s1 = c_perm[t][0], s2 = c_perm[t][1], s3 = c_perm[t][2];
          int v[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
          v[1][s1] = 1;
          v[2][s1] = 1;
          v[2][s2] = 1;
          double gr[4][3] = {};
          gr[0][s1] = -1; gr[1][s1] = 1; gr[1][s2] = -1; gr[2][s2] = 1; gr[2][s3] = -1; gr[3][s3] = 1;
          for (int q = 0; q < 4; ++q) {
            // offset of vertex q from the centre vertex (cube origin = centre + d)
            const int ox = v[q][0] + dx, oy = v[q][1] + dy, oz = v[q][2] + dz;
            const int o = (oz + 1) * 9 + (oy + 1) * 3 + (ox + 1);
            const double gg = gr[m][0] * gr[q][0] + gr[m][1] * gr[q][1] + gr[m][2] * gr[q][2];
            for (int a = 0; a < 3; ++a)
              for (int b = 0; b < 3; ++b) {
                const double G = (a == b) ? vol * gg : 0.0;
                const double S = vol * gr[q][a] * gr[m][b];
                const double D = vol * gr[m][a] * gr[q][b];
                A[FORM_MOD][a][b][o] += G + S - D;
                A[FORM_SYM][a][b][o] += G + S;
                A[FORM_GRAD][a][b][o] += G;
              }
            for (int a = 0; a < 3; ++a) {
              BT[a][o] += -(vol / 4.0) * gr[m][a];
              B[a][o] += -(vol / 4.0) * gr[q][a];
            }
            C[o] += vol * gg;
          }
        }
      }
  double* p = out;
  for (int f = 0; f < 3; ++f)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        for (int o = 0; o < 27; ++o) *p++ = A[f][a][b][o];
  for (int a = 0; a < 3; ++a)
    for (int o = 0; o < 27; ++o) *p++ = BT[a][o];
  for (int a = 0; a < 3; ++a)
    for (int o = 0; o < 27; ++o) *p++ = B[a][o];
  for (int o = 0; o < 27; ++o) *p++ = C[o];
}

// ---- TMA / mbarrier primitives ---------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct StreamArgs {
  double* out;          // y (APPLY), r (RESID), u_out (VEL, 3 fields), T (P1), p (P2)
  const double* aux;    // b (RESID: 4 fields; VEL: f = fields 0..2), g_p (P1), unused
  const double* inU;    // input velocity base (fields 0..2, stride fs)   [list role]
  const double* inP;    // input pressure (APPLY/RESID/VEL/P1) or T (P2)   [list role]
  const int32_t* list;  // irregular rows: owned linear vertex index
  int nlist;
  int list_blocks;      // leading CTAs running the list role
  int kchunk;           // output planes per stream CTA
  unsigned blocks;      // APPLY block mask
  int color, ncolors;   // VEL
  double omega;         // P2
  int ux0, uy0, uz0;    // velocity tensor-map origin (vertex coordinates)
  int skip_list;        // debug (timing only): skip the list role
};

// in-plane offsets of one streamed plane: (0,0) (1,0) (-1,0) (0,1) (0,-1) (1,1) (-1,-1)
__device__ __forceinline__ constexpr int kdx(int q) { return q == 1 || q == 5 ? 1 : (q == 2 || q == 6 ? -1 : 0); }
__device__ __forceinline__ constexpr int kdy(int q) { return q == 3 || q == 5 ? 1 : (q == 4 || q == 6 ? -1 : 0); }
// is (dx,dy,dz) in the 15-point Kuhn pattern (0 or +-d, d in {0,1}^3)?
__device__ __forceinline__ constexpr bool kuhn(int dx, int dy, int dz) {
  return (dx >= 0 && dy >= 0 && dz >= 0) || (dx <= 0 && dy <= 0 && dz <= 0);
}
__device__ __forceinline__ constexpr bool axis_or_centre(int dx, int dy, int dz) {
  return (dx != 0) + (dy != 0) + (dz != 0) <= 1;
}
__device__ __forceinline__ constexpr int oidx(int dx, int dy, int dz) { return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1); }

// accumulators of one output row (unscaled)
struct Acc {
  double A[3], BT[3], B, C;
  __device__ __forceinline__ void zero() {
    A[0] = A[1] = A[2] = BT[0] = BT[1] = BT[2] = B = C = 0.0;
  }
};

template <int FORM, int OP, int DZ>
__device__ __forceinline__ void accumulate(Acc& acc, const double* __restrict__ pl, int base) {
  constexpr bool NEED_U = OP != OP_P1 && OP != OP_P2;   // A, B^T rows
  constexpr bool NEED_P = OP != OP_VEL;                 // B, C rows
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const int dx = kdx(q), dy = kdy(q);
    if (!kuhn(dx, dy, DZ)) continue;
    const int o = oidx(dx, dy, DZ);
    const int s = base + dy * HX + dx;
    if (OP == OP_P2) {
      if (axis_or_centre(dx, dy, DZ)) acc.C += st_C[o] * pl[s];
      continue;
    }
    const double u0 = pl[0 * FST + s], u1 = pl[1 * FST + s], u2 = pl[2 * FST + s];
    const double p = pl[3 * FST + s];
    if (NEED_U) {
      if (FORM == FORM_SYM) {
        const double uu[3] = {u0, u1, u2};
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) acc.A[a] += st_A[FORM_SYM][a][b][o] * uu[b];
      } else if (axis_or_centre(dx, dy, DZ)) {
        const double L = st_A[FORM][0][0][o];
        acc.A[0] += L * u0;
        acc.A[1] += L * u1;
        acc.A[2] += L * u2;
      }
      if (!(dx == 0 && dy == 0 && DZ == 0)) {
        acc.BT[0] += st_BT[0][o] * p;
        acc.BT[1] += st_BT[1][o] * p;
        acc.BT[2] += st_BT[2][o] * p;
      }
    }
    if (NEED_P) {
      if (!(dx == 0 && dy == 0 && DZ == 0)) acc.B += st_B[0][o] * u0 + st_B[1][o] * u1 + st_B[2][o] * u2;
      if (axis_or_centre(dx, dy, DZ)) acc.C += st_C[o] * p;
    }
  }
}

// Truncated-star C row of an isoviscous boundary vertex in unit form:
// (C p)_v = (delta h^3 / (6 mu)) sum_e N_e (p_v - p_e), N_e = number of the 6
// tets around axis edge e that lie inside the cube (cube presence along x:
// X0 = cube at dx = -1 exists (i >= 1), X1 = cube at dx = 0 exists (i <= n-1)).
// Returns s = sum_e N_e p_e and d = sum_e N_e.  pm/p0/pp: planes k-1, k, k+1.
__device__ __forceinline__ void c_trunc(const double* pm, const double* p0, const double* pp, int s, int i,
                                        int j, int k, int n, double& sum, double& diag) {
  const int X0 = i >= 1, X1 = i <= n - 1, Y0 = j >= 1, Y1 = j <= n - 1, Z0 = k >= 1, Z1 = k <= n - 1;
  const int wx = 2 * (Y1 & Z1) + (Y0 & Z1) + (Y1 & Z0) + 2 * (Y0 & Z0);
  const int wy = 2 * (X1 & Z1) + (X0 & Z1) + (X1 & Z0) + 2 * (X0 & Z0);
  const int wz = 2 * (X1 & Y1) + (X0 & Y1) + (X1 & Y0) + 2 * (X0 & Y0);
  double acc = 0.0;
  if (X1 && wx) acc += wx * p0[s + 1];
  if (X0 && wx) acc += wx * p0[s - 1];
  if (Y1 && wy) acc += wy * p0[s + HX];
  if (Y0 && wy) acc += wy * p0[s - HX];
  if (Z1 && wz) acc += wz * pp[s];
  if (Z0 && wz) acc += wz * pm[s];
  sum = acc;
  diag = (double)((X0 + X1) * wx + (Y0 + Y1) * wy + (Z0 + Z1) * wz);
}

// unit B row (sum_o sum_b st_B[b][o] u_b(v+o)) from three staged planes, for the
// face vertices i = n / j = n (SKIPX / SKIPY: offsets with dx = +1 / dy = +1 lie
// outside the staged box; the zero-extended velocity vanishes there)
template <bool SKIPX, bool SKIPY>
__device__ __forceinline__ double b_row_smem(const double* const pl[3], int s) {
  double acc = 0.0;
#pragma unroll
  for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        if (!kuhn(dx, dy, dz) || (dx == 0 && dy == 0 && dz == 0)) continue;
        if ((SKIPX && dx == 1) || (SKIPY && dy == 1)) continue;
        const int o = oidx(dx, dy, dz);
        const double* q = pl[dz + 1] + s + dy * HX + dx;
        acc += st_B[0][o] * q[0 * FST] + st_B[1][o] * q[1 * FST] + st_B[2][o] * q[2 * FST];
      }
  return acc;
}

// finishes a Dirichlet boundary row with an isoviscous star of class `code`
// (velocity rows are 0): Bu = unit B row (OP_APPLY/RESID/P1), planes pl[0..2]
// = k-1, k, k+1 (4-field slots, or 1-field T slots for P2), s = smem position
template <int OP>
__device__ __forceinline__ void finish_boundary(const DGrid& g, const StreamArgs& a, int i, int j, int k,
                                                uint8_t code, double Bu, const double* const pl[3], int s) {
  const int64_t o = vidx(g, i, j, k);
  const double h = g.h;
  constexpr int PF = OP == OP_P2 ? 0 : 3;  // pressure (or T) field within a slot
  double sum, diag;
  c_trunc(pl[0] + PF * FST, pl[1] + PF * FST, pl[2] + PF * FST, s, i, j, k, g.n, sum, diag);
  const double cw = g.delta * h * h * h * c_inv_mu[code] * (1.0 / 6.0);  // per-count edge weight
  const double pv = pl[1][PF * FST + s];
  if (OP == OP_APPLY || OP == OP_RESID) {
    const unsigned blk = OP == OP_APPLY ? a.blocks : BLK_ALL;
    const double yp = ((blk & BLK_B) ? h * h * Bu : 0.0) - ((blk & BLK_C) ? cw * (diag * pv - sum) : 0.0);
    a.out[0 * g.fs + o] = 0.0;
    a.out[1 * g.fs + o] = 0.0;
    a.out[2 * g.fs + o] = 0.0;
    a.out[3 * g.fs + o] = OP == OP_RESID ? __ldg(a.aux + 3 * g.fs + o) - yp : yp;
  } else if (OP == OP_VEL) {
    a.out[0 * g.fs + o] = 0.0;
    a.out[1 * g.fs + o] = 0.0;
    a.out[2 * g.fs + o] = 0.0;
  } else if (OP == OP_P1) {
    const double r = h * h * Bu - cw * (diag * pv - sum) - __ldg(a.aux + o);
    a.out[o] = ((i + j + k) & 1) == 0 ? r / (cw * diag) : r;
  } else {  // P2: pv = T_v; neighbours of a colour-1 vertex are colour 0
    double d = pv;
    if ((i + j + k) & 1) d = (pv + cw * sum) / (cw * diag);
    a.out[o] += a.omega * d;
  }
}

// ---- list role: irregular rows by the element loop -----------------------------
template <int FORM, int OP>
__device__ __forceinline__ void list_row(const DGrid& g, const StreamArgs& a, int i, int j, int k) {
  const int64_t o = vidx(g, i, j, k);
  const bool dir = is_dirichlet(g, i, j, k);
  double y[4], dA[3], dC;
  if (OP == OP_APPLY || OP == OP_RESID) {
    FetchVec fx{a.inU, a.inP};
    row_generic<FORM>(g, i, j, k, fx, OP == OP_APPLY ? a.blocks : BLK_ALL, y, dA, dC);
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      double v = y[f];
      if (OP == OP_RESID) v = (f < 3 && dir) ? 0.0 : __ldg(a.aux + f * g.fs + o) - y[f];
      a.out[f * g.fs + o] = v;
    }
  } else if (OP == OP_VEL) {
    const bool act = ((i + j + k) % a.ncolors) == a.color && !dir;
    if (act) {
      FetchVec fx{a.inU, a.inP};
      row_generic<FORM>(g, i, j, k, fx, BLK_A | BLK_BT, y, dA, dC);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double uc = dir ? 0.0 : __ldg(a.inU + c * g.fs + o);
      a.out[c * g.fs + o] = act ? uc + (__ldg(a.aux + c * g.fs + o) - y[c]) / dA[c] : uc;
    }
  } else if (OP == OP_P1) {
    FetchVec fx{a.inU, a.inP};
    row_generic<FORM>(g, i, j, k, fx, BLK_B | BLK_C, y, dA, dC);
    const double r = y[3] - __ldg(a.aux + o);
    a.out[o] = ((i + j + k) & 1) == 0 ? r / dC : r;
  } else {
    const double T = __ldg(a.inP + o);
    double d = T;
    if ((i + j + k) & 1) {
      FetchRedP fx{a.inP};
      row_generic<FORM>(g, i, j, k, fx, BLK_C, y, dA, dC);
      d = (T + y[3]) / dC;
    }
    a.out[o] += a.omega * d;
  }
}

template <int FORM, int OP>
__device__ __noinline__ void list_role(const DGrid& g, const StreamArgs& a) {
  const int e = blockIdx.x * NT + threadIdx.x;
  if (e >= a.nlist || a.skip_list) return;
  const int t = a.list[e];
  const int nx = g.n + 1;
  const int k = g.z0 + t / (nx * nx);
  const int r = t % (nx * nx);
  list_row<FORM, OP>(g, a, r % nx, r / nx, k);
}

// ---- stream role ----------------------------------------------------------------
template <int FORM, int OP>
__global__ void __launch_bounds__(NT, 2)
    k_stream(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapP, DGrid g,
             StreamArgs a) {
  if ((int)blockIdx.x < a.list_blocks) {
    list_role<FORM, OP>(g, a);
    return;
  }
  constexpr int NF = OP == OP_P2 ? 1 : 4;
  constexpr uint32_t TX_BYTES = NF * PLANE * sizeof(double);  // bytes landed per plane
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem_raw =
      smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);  // 1 KB aligned TMA destinations
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + RING * NF * FST * sizeof(double));

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int ntx = g.n / TX;
  const int tiles = ntx * (g.n / TY);
  const int sb = blockIdx.x - a.list_blocks;
  const int tile = sb % tiles, chunk = sb / tiles;   // chunk-major: neighbours share L2
  const int i0 = (tile % ntx) * TX, j0 = (tile / ntx) * TY;
  const int kb = g.z0 + chunk * a.kchunk;
  const int ke = min(kb + a.kchunk, g.z0 + g.nzl);
  if (kb >= ke) return;
  const int M = ke - kb + 2;  // planes kb-1 .. ke
  const int kb1 = kb - 1;
  const bool last_x = i0 + TX == g.n, last_y = j0 + TY == g.n;
  const int i = i0 + tx, j = j0 + ty;
  const int base = (ty + 1) * HX + (tx + 1);
  const double h = g.h;
  const double sA = h, sB = h * h, sC = g.delta * h * h * h;  // times mu / 1 / 1/mu
  // extra face rows: (n, j) for the last lane of last-x tiles, (i, n) for the
  // last warp of last-y tiles, (n, n) for the last thread of the corner tile
  const bool ex_x = last_x && tx == TX - 1, ex_y = last_y && ty == TY - 1, ex_c = ex_x && ex_y;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int m) {
    if (m >= M) return;
    const int s = m % RING;
    const int P = kb1 + m;
    fence_proxy_async();
    mbar_expect_tx(&bars[s], TX_BYTES);
    double* dst = ring + s * NF * FST;
    if (NF == 4) {
      for (int f = 0; f < 3; ++f)
        tma_load_4d(dst + f * FST, &mapU, &bars[s], i0 - 1 - a.ux0, j0 - 1 - a.uy0, P - a.uz0, f);
      tma_load_4d(dst + 3 * FST, &mapP, &bars[s], i0, j0, P - g.z0 + 1, 0);
    } else {
      tma_load_4d(dst, &mapP, &bars[s], i0, j0, P - g.z0 + 1, 0);
    }
  };
  if (threadIdx.x == 0)
    for (int m = 0; m < PREF; ++m) issue(m);

  Acc acc0, acc1, acc2;  // outputs P-1, P, P+1
  acc0.zero();
  acc1.zero();
  acc2.zero();

  for (int m = 0; m < M; ++m) {
    const int P = kb1 + m;
    const int k = P - 1;  // output finished in this iteration
    const bool fin = m >= 2;
    // early loads of per-output data (codes, own auxiliary values)
    uint8_t code = CODE_IRREGULAR, code_x = CODE_IRREGULAR, code_y = CODE_IRREGULAR, code_c = CODE_IRREGULAR;
    double aux[4] = {0, 0, 0, 0};
    if (fin) {
      const int64_t o = vidx(g, i, j, k);
      code = __ldg(g.code + o);
      if (ex_x) code_x = __ldg(g.code + o + 1);
      if (ex_y) code_y = __ldg(g.code + o + g.px);
      if (ex_c) code_c = __ldg(g.code + o + g.px + 1);
      if (!(code & 0x80)) {
        if (OP == OP_RESID) {
#pragma unroll
          for (int f = 0; f < 4; ++f) aux[f] = __ldg(a.aux + f * g.fs + o);
        } else if (OP == OP_VEL) {
#pragma unroll
          for (int f = 0; f < 3; ++f) aux[f] = __ldg(a.aux + f * g.fs + o);
        } else if (OP == OP_P1) {
          aux[3] = __ldg(a.aux + o);
        } else if (OP == OP_P2) {
          aux[3] = a.out[o];
        }
      }
    }
    const int s = m % RING;
    mbar_wait(&bars[s], (m / RING) & 1);
    const double* pl = ring + s * NF * FST;
    accumulate<FORM, OP, 1>(acc0, pl, base);   // plane P is output P-1's z+1 plane
    accumulate<FORM, OP, 0>(acc1, pl, base);
    accumulate<FORM, OP, -1>(acc2, pl, base);

    if (fin) {
      const int64_t o = vidx(g, i, j, k);
      const double* pls[3] = {ring + ((m - 2) % RING) * NF * FST, ring + ((m - 1) % RING) * NF * FST, pl};
      if (!(code & 0x80)) {
        const bool interior = i > 0 && j > 0 && k > 0 && k < g.n;
        if (!interior) {
          finish_boundary<OP>(g, a, i, j, k, code, acc0.B, pls, base);
        } else {
          const double mu = c_mu[code], imu = c_inv_mu[code];
          if (OP == OP_APPLY || OP == OP_RESID) {
            double y[4];
#pragma unroll
            for (int c = 0; c < 3; ++c)
              y[c] = ((a.blocks & BLK_A) ? mu * sA * acc0.A[c] : 0.0) + ((a.blocks & BLK_BT) ? sB * acc0.BT[c] : 0.0);
            y[3] = ((a.blocks & BLK_B) ? sB * acc0.B : 0.0) - ((a.blocks & BLK_C) ? sC * imu * acc0.C : 0.0);
#pragma unroll
            for (int f = 0; f < 4; ++f) a.out[f * g.fs + o] = OP == OP_RESID ? aux[f] - y[f] : y[f];
          } else if (OP == OP_VEL) {
            const bool act = ((i + j + k) % a.ncolors) == a.color;
            const double* cpl = pls[1];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double uc = cpl[c * FST + base];
              double v = uc;
              if (act) {
                const double y = mu * sA * acc0.A[c] + sB * acc0.BT[c];
                v = uc + (aux[c] - y) / (mu * sA * st_A[FORM][c][c][13]);
              }
              a.out[c * g.fs + o] = v;
            }
          } else if (OP == OP_P1) {
            const double r = sB * acc0.B - sC * imu * acc0.C - aux[3];
            a.out[o] = ((i + j + k) & 1) == 0 ? r / (sC * imu * st_C[13]) : r;
          } else {  // P2: acc0.C holds sum_o C[o] T (including the centre)
            const double T = pls[1][base];
            double d = T;
            if ((i + j + k) & 1) {
              const double off = acc0.C - st_C[13] * T;  // neighbours only (all colour 0)
              d = (T - sC * imu * off) / (sC * imu * st_C[13]);
            }
            a.out[o] = aux[3] + a.omega * d;
          }
        }
      }
      // face rows i = n, j = n (Dirichlet with an isoviscous star, else list rows)
      if (ex_x && !(code_x & 0x80)) {
        const double Bu = (OP == OP_P2 || OP == OP_VEL) ? 0.0 : b_row_smem<true, false>(pls, base + 1);
        finish_boundary<OP>(g, a, g.n, j, k, code_x, Bu, pls, base + 1);
      }
      if (ex_y && !(code_y & 0x80)) {
        const double Bu = (OP == OP_P2 || OP == OP_VEL) ? 0.0 : b_row_smem<false, true>(pls, base + HX);
        finish_boundary<OP>(g, a, i, g.n, k, code_y, Bu, pls, base + HX);
      }
      if (ex_c && !(code_c & 0x80)) {
        const double Bu = (OP == OP_P2 || OP == OP_VEL) ? 0.0 : b_row_smem<true, true>(pls, base + HX + 1);
        finish_boundary<OP>(g, a, g.n, g.n, k, code_c, Bu, pls, base + HX + 1);
      }
    }
    __syncthreads();  // slot of plane m-2 is free for plane m+PREF
    if (threadIdx.x == 0) issue(m + PREF);
    acc0 = acc1;
    acc1 = acc2;
    acc2.zero();
  }
}

// ---- host side --------------------------------------------------------------

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled encoder() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

// 4-D map (x, y, z-plane, field) over vertices [x0, x1] x [y0, y1] x [z0v, z1v]
// of a level vector `base` (field 0), box = one staged plane of one field.
inline bool make_map(CUtensorMap* map, const double* base, const DGrid& g, int nfields, int x0, int x1, int y0,
                     int y1, int z0v, int z1v) {
  PFN_encodeTiled enc = encoder();
  if (!enc) return false;
  const double* origin = base + vidx_host(g, x0, y0, z0v);
  cuuint64_t dims[4] = {(cuuint64_t)(x1 - x0 + 1), (cuuint64_t)(y1 - y0 + 1), (cuuint64_t)(z1v - z0v + 1),
                        (cuuint64_t)nfields};
  cuuint64_t strides[3] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.py * 8, (cuuint64_t)g.fs * 8};
  cuuint32_t box[4] = {HX, HY, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)origin, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool tiled_supported(int n) { return n >= 64 && n % TX == 0 && n % TY == 0 && encoder() != nullptr; }

inline bool assemble_stencils(cudaStream_t st) {
  static bool done = false;
  if (done) return true;
  double* d = nullptr;
  const size_t cnt = 3 * 9 * 27 + 3 * 27 + 3 * 27 + 27;
  if (cudaMalloc(&d, cnt * sizeof(double)) != cudaSuccess) return false;
  k_assemble_stencils<<<1, 32, 0, st>>>(d);
  size_t off = 0;
  bool ok = cudaMemcpyToSymbolAsync(st_A, d + off, sizeof(st_A), 0, cudaMemcpyDeviceToDevice, st) == cudaSuccess;
  off += 3 * 9 * 27;
  ok &= cudaMemcpyToSymbolAsync(st_BT, d + off, sizeof(st_BT), 0, cudaMemcpyDeviceToDevice, st) == cudaSuccess;
  off += 3 * 27;
  ok &= cudaMemcpyToSymbolAsync(st_B, d + off, sizeof(st_B), 0, cudaMemcpyDeviceToDevice, st) == cudaSuccess;
  off += 3 * 27;
  ok &= cudaMemcpyToSymbolAsync(st_C, d + off, sizeof(st_C), 0, cudaMemcpyDeviceToDevice, st) == cudaSuccess;
  ok &= cudaStreamSynchronize(st) == cudaSuccess;
  cudaFree(d);
  done = ok;
  return ok;
}

inline size_t stream_smem(int op) {
  const int NF = op == OP_P2 ? 1 : 4;
  return 1024 + RING * NF * FST * sizeof(double) + RING * sizeof(uint64_t);
}

// the irregular-row list of a level (built by stk_assemble)
struct ListView {
  const int32_t* list;
  int n;
};

template <int FORM, int OP>
bool launch_stream_t(const DGrid& g, const double* inU, const double* inP, const ListView& lv,
                     const StreamArgs& a0, cudaStream_t st) {
  const unsigned dm = g.dirmask;
  StreamArgs a = a0;
  // velocity map: one vertex inside every Dirichlet face (OOB zero fill = u_D = 0)
  a.ux0 = (dm & 1u) ? 1 : -1;
  a.uy0 = (dm & 4u) ? 1 : -1;
  const int ux1 = (dm & 2u) ? g.n - 1 : g.n, uy1 = (dm & 8u) ? g.n - 1 : g.n;
  a.uz0 = std::max(g.z0 - 1, (dm & 16u) ? 1 : 0);
  const int uz1 = std::min(g.z0 + g.nzl, (dm & 32u) ? g.n - 1 : g.n);
  CUtensorMap mU, mP;
  if (OP != OP_P2) {
    if (uz1 < a.uz0) return false;
    if (!make_map(&mU, inU, g, 3, a.ux0, ux1, a.uy0, uy1, a.uz0, uz1)) return false;
  }
  // pressure (or T) map: the whole stored slab incl. ghost frame and halo planes
  if (!make_map(&mP, inP, g, 1, -1, g.n, -1, g.n, g.z0 - 1, g.z0 + g.nzl)) return false;
  if (OP == OP_P2) mU = mP;
  const size_t sm = stream_smem(OP);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_stream<FORM, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
      return false;
    attr = true;
  }
  const int tiles = (g.n / TX) * (g.n / TY);
  static const int kchunk_env = getenv("STK_KCHUNK") ? atoi(getenv("STK_KCHUNK")) : 0;
  int kc = kchunk_env > 0 ? kchunk_env : 8;
  kc = std::max(1, std::min(kc, g.nzl));
  const int chunks = (g.nzl + kc - 1) / kc;
  a.kchunk = kc;
  a.inU = inU;
  a.inP = inP;
  a.list = lv.list;
  a.nlist = lv.n;
  a.list_blocks = (lv.n + NT - 1) / NT;
  static const int skip_list = getenv("STK_SKIP_IRR") ? atoi(getenv("STK_SKIP_IRR")) : 0;
  a.skip_list = skip_list;
  k_stream<FORM, OP><<<dim3(a.list_blocks + tiles * chunks), NT, sm, st>>>(mU, mP, g, a);
  return true;
}

template <int OP>
bool launch_stream(int form, const DGrid& g, const double* inU, const double* inP, const ListView& lv,
                   const StreamArgs& a, cudaStream_t st) {
  switch (form) {
    case FORM_MOD: return launch_stream_t<FORM_MOD, OP>(g, inU, inP, lv, a, st);
    case FORM_SYM: return launch_stream_t<FORM_SYM, OP>(g, inU, inP, lv, a, st);
    default: return launch_stream_t<FORM_GRAD, OP>(g, inU, inP, lv, a, st);
  }
}

inline bool launch_apply_tiled(int form, DGrid g, const ListView& lv, const double* x, double* y, unsigned blocks,
                               cudaStream_t st) {
  StreamArgs a{};
  a.out = y;
  a.blocks = blocks;
  return launch_stream<OP_APPLY>(form, g, x, x + 3 * g.fs, lv, a, st);
}
inline bool launch_residual_tiled(int form, DGrid g, const ListView& lv, const double* x, const double* b, double* r,
                                  cudaStream_t st) {
  StreamArgs a{};
  a.out = r;
  a.aux = b;
  a.blocks = BLK_ALL;
  return launch_stream<OP_RESID>(form, g, x, x + 3 * g.fs, lv, a, st);
}
inline bool launch_vel_pass_tiled(int form, DGrid g, const ListView& lv, const double* uin, const double* p,
                                  const double* b, double* uout, int color, int ncolors, cudaStream_t st) {
  StreamArgs a{};
  a.out = uout;
  a.aux = b;
  a.color = color;
  a.ncolors = ncolors;
  return launch_stream<OP_VEL>(form, g, uin, p, lv, a, st);
}
inline bool launch_p_pass1_tiled(int form, DGrid g, const ListView& lv, const double* x, const double* gp, double* T,
                                 cudaStream_t st) {
  StreamArgs a{};
  a.out = T;
  a.aux = gp;
  return launch_stream<OP_P1>(form, g, x, x + 3 * g.fs, lv, a, st);
}
inline bool launch_p_pass2_tiled(int form, DGrid g, const ListView& lv, const double* T, double* p, double omega,
                                 cudaStream_t st) {
  StreamArgs a{};
  a.out = p;
  a.omega = omega;
  return launch_stream<OP_P2>(form, g, T, T, lv, a, st);
}

}  // namespace stk
