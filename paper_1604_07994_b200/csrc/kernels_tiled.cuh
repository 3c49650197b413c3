// Tiled constant-stencil kernels for levels with n >= 64 (the hot path).
//
// Design:
//  * List rows (interface Gamma_12, the traction boundary Gamma_F, vertices
//    touching both kinds of faces) are evaluated by a second kernel, k_listx:
//    16 lanes per row over the row's explicit 4x4-block stencils (assembled
//    once per level from the element loop), reading the input from
//    global memory (L2).  The two kernels write disjoint rows; k_listx runs on
//    a side stream forked from (and joined back into) the caller's stream, and
//    the stream kernels' register caps leave room for one of its CTAs per SM
//    (STK_LIST_EXPLICIT=0: the per-thread element loop k_list instead;
//    STK_LIST_FORK=0: serial).
//  * A stream CTA owns a TX x TY column tile (i in [i0, i0+TX), j in
//    [j0, j0+TY), i0+TX <= n) and a chunk of z-planes.  Each plane of the input
//    fields, with a 1-vertex xy halo, is staged in shared memory by TMA boxes
//    (cp.async.bulk.tensor.4d + mbarrier complete_tx), PREF planes ahead, in a
//    ring of PREF+2 slots.  One __syncthreads per plane.  CTAs are persistent
//    (one per resident slot) and take items (tile, z-chunk) round robin.
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

#include <cmath>
#include <cstdlib>
#include <vector>

#include "stk_common.cuh"

namespace stk {

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int HX = TX + 2, HY = TY + 2, PLANE = HX * HY;
// shared-memory stride of one staged field plane: 128-byte aligned TMA destinations
constexpr int FST = ((PLANE + 15) / 16) * 16;
constexpr int PREF = 3, RING = PREF + 2;
// STK_MU_SMEM=1: the per-class (mu, 1/mu) table is copied to shared memory at kernel
// start; the row finish reads it from there (a ~30-cycle LDS) instead of two dependent
// global loads behind the code byte (ncu: 0.6-2.0 long-scoreboard stall cycles per issue).
#ifndef STK_MU_SMEM
#define STK_MU_SMEM 0
#endif
__device__ __forceinline__ double tab_ld(const double* mt, int idx) {
#if STK_MU_SMEM
  return mt[idx];
#else
  return __ldg(mt + idx);
#endif
}
// per-row auxiliary fields, prefetched one row ahead by cp.async into a per-thread
// double buffer: RESID b (4), VEL f (3), P1 g (1), P2 own p (1)
__host__ __device__ constexpr int n_aux(int op) { return op == 1 ? 4 : op == 2 ? 3 : (op == 3 || op == 4) ? 1 : 0; }
// doubles per ring slot: staged fields (with halo)
__host__ __device__ constexpr int slot_doubles(int op) { return (op == 4 ? 1 : 4) * FST; }


// Integer unit stencils of an interior vertex (h = 1, mu = 1, delta = 1), by
// the element sum over the 24 tets of its star, evaluated at compile time:
//   kind 0: 6 A_form[a][b](o), kind 1: 24 B^T[a](o), kind 2: 24 B[b](o), kind 3: 6 C(o)
// (the factors 6 and 24 make every entry an integer: |T| = 1/6, B = -|T|/4 grad).
// A regular row of class k scales them by mu_k h / 6, h^2 / 24, h^2 / 24 and
// delta h^3 / (6 mu_k) ("interior stencils can be pre-computed").
// k_assemble_stencils sums the same element matrices at run time in floating
// point and stk_assemble checks the two agree (k_check_stencils).
__host__ __device__ constexpr int kst(int kind, int form, int a, int b, int dx, int dy, int dz, int cmask = 0xFF) {
  int s = 0;
  for (int cz = -1; cz <= 0; ++cz)
    for (int cy = -1; cy <= 0; ++cy)
      for (int cx = -1; cx <= 0; ++cx) {
        const int corner = (-cx) | ((-cy) << 1) | ((-cz) << 2);
        if (!((cmask >> corner) & 1)) continue;  // cube absent (outside the domain)
        for (int t = 0; t < 6; ++t) {
          const int m = kcorner(corner, t);
          if (m < 0) continue;
          int gr[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          const int s1 = kperm(t, 0), s2 = kperm(t, 1), s3 = kperm(t, 2);
          gr[0][s1] = -1; gr[1][s1] = 1; gr[1][s2] = -1; gr[2][s2] = 1; gr[2][s3] = -1; gr[3][s3] = 1;
          for (int q = 0; q < 4; ++q) {
            const int c = ktet_corner(t, q);
            if ((c & 1) + cx != dx || ((c >> 1) & 1) + cy != dy || (c >> 2) + cz != dz) continue;
            const int gg = gr[m][0] * gr[q][0] + gr[m][1] * gr[q][1] + gr[m][2] * gr[q][2];
            if (kind == 0) {
              const int G = (a == b) ? gg : 0, S = gr[q][a] * gr[m][b], D = gr[m][a] * gr[q][b];
              s += form == FORM_MOD ? G + S - D : form == FORM_SYM ? G + S : G;
            } else if (kind == 1) {
              s -= gr[m][a];
            } else if (kind == 2) {
              s -= gr[q][b];
            } else {
              s += gg;
            }
          }
        }
      }
  return s;
}
template <int KIND, int FORM, int A, int B, int DX, int DY, int DZ>
struct KS {
  static constexpr double v = (double)kst(KIND, FORM, A, B, DX, DY, DZ);
};
// truncated stencils of a vertex on the top face z = 1 (only the 4 cubes below
// it, own corners 4..7, lie in the domain): the rows of an isoviscous traction
// top-face vertex (Gamma_F), evaluated by the same element sum
constexpr int KTOP_MASK = 0xF0;
template <int KIND, int FORM, int A, int B, int DX, int DY, int DZ>
struct KT {
  static constexpr double v = (double)kst(KIND, FORM, A, B, DX, DY, DZ, KTOP_MASK);
};
constexpr uint8_t CODE_TOP = 0x40;  // code bit: isoviscous traction top-face row (class in bits 0..5)
// closed forms of SURVEY App. A.2 (compile-time checks of the element sums)
constexpr bool kst_closed_forms_hold() {
  for (int o = 0; o < 27; ++o) {
    const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
    const int nax = (dx != 0) + (dy != 0) + (dz != 0);
    const int lap = nax == 0 ? 36 : nax == 1 ? -6 : 0;  // 6 x (6, -1, 0)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        if (kst(0, FORM_GRAD, a, b, dx, dy, dz) != (a == b ? lap : 0)) return false;
        if (kst(0, FORM_MOD, a, b, dx, dy, dz) != (a == b ? lap : 0)) return false;  // cross part 0
      }
    if (kst(3, 0, 0, 0, dx, dy, dz) != lap) return false;
  }
  // (Bu)(i) = h^2/24 sum_b sum_{d in D+} beta^b_d (u_b(i-d) - u_b(i+d)), beta = 6 (d = e_b),
  // 2 (d_b = 1), -2 (d_b = 0); B^T p pairs p(i+d) - p(i-d) with the same beta
  return kst(2, 0, 0, 0, 1, 0, 0) == -6 && kst(2, 0, 0, 1, 1, 0, 0) == 2 && kst(2, 0, 0, 0, 1, 1, 0) == -2 &&
         kst(2, 0, 0, 0, -1, -1, -1) == 2 && kst(1, 0, 0, 0, 1, 0, 0) == 6 && kst(2, 0, 0, 0, 0, 0, 0) == 0;
}
static_assert(kst_closed_forms_hold(), "Kuhn unit stencils disagree with the closed forms");

// run-time stencils assembled by k_assemble_stencils (floating point), checked
// against kst by k_check_stencils
__constant__ double st_A[3][3][3][27];  // [form][a][b][o]
__constant__ double st_BT[3][27];       // velocity row a, pressure column
__constant__ double st_B[3][27];        // pressure row, velocity column b
__constant__ double st_C[27];

enum { OP_APPLY = 0, OP_RESID = 1, OP_VEL = 2, OP_P1 = 3, OP_P2 = 4 };
#ifndef STK_TMA_FENCE
#define STK_TMA_FENCE 1
#endif
#ifndef STK_TMA_PREFETCH
#define STK_TMA_PREFETCH 0
#endif


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
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct StreamArgs {
  double* out;          // y (APPLY), r (RESID), u_out (VEL, 3 fields), T (P1), p (P2)
  const double* aux;    // b (RESID: 4 fields; VEL: f = fields 0..2), g_p (P1), unused
  const double* inU;    // input velocity base (fields 0..2, stride fs)   [list role]
  const double* inP;    // input pressure (APPLY/RESID/VEL/P1) or T (P2)   [list role]
  const int32_t* list;  // irregular rows: owned linear vertex index
  int nlist;
  int kchunk;           // output planes per stream CTA
  unsigned blocks;      // APPLY block mask
  int color, ncolors;   // VEL
  double omega;         // P2
  int ux0, uy0, uz0;    // velocity tensor-map origin (vertex coordinates)
  int inplace;          // VEL: out == input velocity; only the active colour's stream rows are written,
                        // list and traction-face rows go to cbuf (k_listx) and are scattered after
  double* cbuf;         // VEL list rows: results [row][3] instead of out (nullptr: write out)
  unsigned long long* trace;  // debug (STK_STREAM_TRACE): per-CTA cycle counters, else nullptr
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

// accumulators of one output row, in integer-stencil units (6A, 24B^T, 24B, 6C)
struct Acc {
  double A[3], BT[3], B, C;
  __device__ __forceinline__ void zero() {
    A[0] = A[1] = A[2] = BT[0] = BT[1] = BT[2] = B = C = 0.0;
  }
};

// contribution of staged in-plane point Q (offset (kdx(Q), kdy(Q)) from the
// output column, plane offset DZ from the output row) to one output row, from
// the point's values already in registers (u0, u1, u2, p)
template <int FORM, int OP, int DZ, int Q>
__device__ __forceinline__ void acc_v(Acc& acc, double u0, double u1, double u2, double p) {
  constexpr int dx = kdx(Q), dy = kdy(Q);
  if constexpr (kuhn(dx, dy, DZ)) {
    constexpr bool NEED_U = OP != OP_P1 && OP != OP_P2;  // A, B^T rows
    constexpr bool NEED_P = OP != OP_VEL;                // B, C rows
    constexpr double kC = KS<3, 0, 0, 0, dx, dy, DZ>::v;
    if constexpr (OP == OP_P2) {
      if constexpr (kC != 0.0) acc.C = fma(kC, p, acc.C);
    } else {
      if constexpr (NEED_U) {
        if constexpr (FORM == FORM_SYM) {
          acc.A[0] = fma(KS<0, FORM_SYM, 0, 0, dx, dy, DZ>::v, u0, acc.A[0]);
          acc.A[0] = fma(KS<0, FORM_SYM, 0, 1, dx, dy, DZ>::v, u1, acc.A[0]);
          acc.A[0] = fma(KS<0, FORM_SYM, 0, 2, dx, dy, DZ>::v, u2, acc.A[0]);
          acc.A[1] = fma(KS<0, FORM_SYM, 1, 0, dx, dy, DZ>::v, u0, acc.A[1]);
          acc.A[1] = fma(KS<0, FORM_SYM, 1, 1, dx, dy, DZ>::v, u1, acc.A[1]);
          acc.A[1] = fma(KS<0, FORM_SYM, 1, 2, dx, dy, DZ>::v, u2, acc.A[1]);
          acc.A[2] = fma(KS<0, FORM_SYM, 2, 0, dx, dy, DZ>::v, u0, acc.A[2]);
          acc.A[2] = fma(KS<0, FORM_SYM, 2, 1, dx, dy, DZ>::v, u1, acc.A[2]);
          acc.A[2] = fma(KS<0, FORM_SYM, 2, 2, dx, dy, DZ>::v, u2, acc.A[2]);
        } else {
          constexpr double kA = KS<0, FORM_GRAD, 0, 0, dx, dy, DZ>::v;  // = mod on regular rows
          if constexpr (kA != 0.0) {
            acc.A[0] = fma(kA, u0, acc.A[0]);
            acc.A[1] = fma(kA, u1, acc.A[1]);
            acc.A[2] = fma(kA, u2, acc.A[2]);
          }
        }
        constexpr double kT0 = KS<1, 0, 0, 0, dx, dy, DZ>::v, kT1 = KS<1, 0, 1, 0, dx, dy, DZ>::v,
                         kT2 = KS<1, 0, 2, 0, dx, dy, DZ>::v;
        if constexpr (kT0 != 0.0) acc.BT[0] = fma(kT0, p, acc.BT[0]);
        if constexpr (kT1 != 0.0) acc.BT[1] = fma(kT1, p, acc.BT[1]);
        if constexpr (kT2 != 0.0) acc.BT[2] = fma(kT2, p, acc.BT[2]);
      }
      if constexpr (NEED_P) {
        constexpr double kB0 = KS<2, 0, 0, 0, dx, dy, DZ>::v, kB1 = KS<2, 0, 0, 1, dx, dy, DZ>::v,
                         kB2 = KS<2, 0, 0, 2, dx, dy, DZ>::v;
        if constexpr (kB0 != 0.0) acc.B = fma(kB0, u0, acc.B);
        if constexpr (kB1 != 0.0) acc.B = fma(kB1, u1, acc.B);
        if constexpr (kB2 != 0.0) acc.B = fma(kB2, u2, acc.B);
        if constexpr (kC != 0.0) acc.C = fma(kC, p, acc.C);
      }
    }
  }
}

// point Q of a landed plane: its values are read from shared memory ONCE and
// added to the outputs one plane below (acc0, DZ = +1), in the plane (acc1, DZ = 0)
// and one plane above (acc2, DZ = -1); MASK: bit0 acc0, bit1 acc1, bit2 acc2
template <int FORM, int OP, int Q, int MASK>
__device__ __forceinline__ void point3(Acc& acc0, Acc& acc1, Acc& acc2, const double* __restrict__ pl, int base) {
  constexpr int dx = kdx(Q), dy = kdy(Q);
  constexpr bool U0 = (MASK & 1) && kuhn(dx, dy, 1), U1 = (MASK & 2) && kuhn(dx, dy, 0), U2 = (MASK & 4) && kuhn(dx, dy, -1);
  if constexpr (U0 || U1 || U2) {
    const int s = base + dy * HX + dx;
    double u0 = 0.0, u1 = 0.0, u2 = 0.0, p;
    if constexpr (OP == OP_P2) {
      p = pl[s];
    } else {
      u0 = pl[s];
      u1 = pl[FST + s];
      u2 = pl[2 * FST + s];
      p = pl[3 * FST + s];
    }
    if constexpr (U0) acc_v<FORM, OP, 1, Q>(acc0, u0, u1, u2, p);
    if constexpr (U1) acc_v<FORM, OP, 0, Q>(acc1, u0, u1, u2, p);
    if constexpr (U2) acc_v<FORM, OP, -1, Q>(acc2, u0, u1, u2, p);
  }
}
template <int FORM, int OP, int MASK>
__device__ __forceinline__ void accumulate3(Acc& acc0, Acc& acc1, Acc& acc2, const double* __restrict__ pl, int base) {
  point3<FORM, OP, 0, MASK>(acc0, acc1, acc2, pl, base);
  point3<FORM, OP, 1, MASK>(acc0, acc1, acc2, pl, base);
  point3<FORM, OP, 2, MASK>(acc0, acc1, acc2, pl, base);
  point3<FORM, OP, 3, MASK>(acc0, acc1, acc2, pl, base);
  point3<FORM, OP, 4, MASK>(acc0, acc1, acc2, pl, base);
  point3<FORM, OP, 5, MASK>(acc0, acc1, acc2, pl, base);
  point3<FORM, OP, 6, MASK>(acc0, acc1, acc2, pl, base);
}
// single-output form (prologue planes)
template <int FORM, int OP, int DZ>
__device__ __forceinline__ void accumulate(Acc& acc, const double* __restrict__ pl, int base) {
  if constexpr (DZ == 1) accumulate3<FORM, OP, 1>(acc, acc, acc, pl, base);
  else if constexpr (DZ == 0) accumulate3<FORM, OP, 2>(acc, acc, acc, pl, base);
  else accumulate3<FORM, OP, 4>(acc, acc, acc, pl, base);
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

// 24 x unit B row (sum_o sum_b kst(2,b,o) u_b(v+o)) from three staged planes, for the
// face vertices i = n / j = n (SKIPX / SKIPY: offsets with dx = +1 / dy = +1 lie
// outside the staged box; the zero-extended velocity vanishes there)
template <int DX, int DY, int DZ, bool SKIPX, bool SKIPY>
__device__ __forceinline__ void b_off(double& acc, const double* const pl[3], int s) {
  if constexpr (kuhn(DX, DY, DZ) && !(DX == 0 && DY == 0 && DZ == 0) && !(SKIPX && DX == 1) && !(SKIPY && DY == 1)) {
    const double* q = pl[DZ + 1] + s + DY * HX + DX;
    acc = fma(KS<2, 0, 0, 0, DX, DY, DZ>::v, q[0 * FST], acc);
    acc = fma(KS<2, 0, 0, 1, DX, DY, DZ>::v, q[1 * FST], acc);
    acc = fma(KS<2, 0, 0, 2, DX, DY, DZ>::v, q[2 * FST], acc);
  }
}
template <int DZ, bool SKIPX, bool SKIPY>
__device__ __forceinline__ void b_plane(double& acc, const double* const pl[3], int s) {
  b_off<-1, -1, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<0, -1, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<1, -1, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<-1, 0, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<0, 0, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<1, 0, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<-1, 1, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<0, 1, DZ, SKIPX, SKIPY>(acc, pl, s);
  b_off<1, 1, DZ, SKIPX, SKIPY>(acc, pl, s);
}
template <bool SKIPX, bool SKIPY>
__device__ __forceinline__ double b_row_smem(const double* const pl[3], int s) {
  double acc = 0.0;
  b_plane<-1, SKIPX, SKIPY>(acc, pl, s);
  b_plane<0, SKIPX, SKIPY>(acc, pl, s);
  b_plane<1, SKIPX, SKIPY>(acc, pl, s);
  return acc;
}

// finishes a Dirichlet boundary row with an isoviscous star of class `code`
// (velocity rows are 0): Bu = 24 x unit B row (OP_APPLY/RESID/P1), planes pl[0..2]
// = k-1, k, k+1 (4-field slots, or 1-field T slots for P2), s = smem position
template <int OP>
__device__ __forceinline__ void finish_boundary(const DGrid& g, const StreamArgs& a, int i, int j, int k,
                                                uint8_t code, double Bu, const double* const pl[3], int s,
                                                const double* mt) {
  const int64_t o = vidx(g, i, j, k);
  const double h = g.h;
  constexpr int PF = OP == OP_P2 ? 0 : 3;  // pressure (or T) field within a slot
  double sum, diag;
  c_trunc(pl[0] + PF * FST, pl[1] + PF * FST, pl[2] + PF * FST, s, i, j, k, g.n, sum, diag);
  const double cw = g.delta * h * h * h * tab_ld(mt, 256 + code) * (1.0 / 6.0);  // per-count edge weight
  const double pv = pl[1][PF * FST + s];
  if (OP == OP_APPLY || OP == OP_RESID) {
    const unsigned blk = OP == OP_APPLY ? a.blocks : BLK_ALL;
    const double yp = ((blk & BLK_B) ? (h * h / 24.0) * Bu : 0.0) - ((blk & BLK_C) ? cw * (diag * pv - sum) : 0.0);
    a.out[0 * g.fs + o] = 0.0;
    a.out[1 * g.fs + o] = 0.0;
    a.out[2 * g.fs + o] = 0.0;
    a.out[3 * g.fs + o] = OP == OP_RESID ? __ldg(a.aux + 3 * g.fs + o) - yp : yp;
  } else if (OP == OP_VEL) {
    a.out[0 * g.fs + o] = 0.0;
    a.out[1 * g.fs + o] = 0.0;
    a.out[2 * g.fs + o] = 0.0;
  } else if (OP == OP_P1) {
    const double r = (h * h / 24.0) * Bu - cw * (diag * pv - sum) - __ldg(a.aux + o);
    a.out[o] = ((i + j + k) & 1) == 0 ? r / (cw * diag) : r;
  } else {  // P2: pv = T_v; neighbours of a colour-1 vertex are colour 0
    double d = pv;
    if ((i + j + k) & 1) d = (pv + cw * sum) / (cw * diag);
    a.out[o] += a.omega * d;
  }
}

// ---- list rows: irregular rows by the element loop, one row per thread -----------
template <int FORM, int OP>
__device__ __forceinline__ void list_row(const DGrid& g, const StreamArgs& a, int i, int j, int k) {
  const int64_t o = vidx(g, i, j, k);
  const unsigned em = elim(g, i, j, k);
  double y[4], dA[3], dC;
  if (OP == OP_APPLY || OP == OP_RESID) {
    row_list<FORM, false>(g, i, j, k, a.inU, a.inP, OP == OP_APPLY ? a.blocks : BLK_ALL, y, dA, dC);
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      double v = y[f];
      if (OP == OP_RESID) v = ((em >> f) & 1u) ? 0.0 : __ldg(a.aux + f * g.fs + o) - y[f];
      a.out[f * g.fs + o] = v;
    }
  } else if (OP == OP_VEL) {
    const bool act = ((i + j + k) & (a.ncolors - 1)) == a.color && em != 7u;
    if (act) row_list<FORM, false>(g, i, j, k, a.inU, a.inP, BLK_A | BLK_BT, y, dA, dC);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const bool ec = (em >> c) & 1u;
      const double uc = ec ? 0.0 : __ldg(a.inU + c * g.fs + o);
      a.out[c * g.fs + o] = (act && !ec) ? uc + (__ldg(a.aux + c * g.fs + o) - y[c]) / dA[c] : uc;
    }
  } else if (OP == OP_P1) {
    row_list<FORM, false>(g, i, j, k, a.inU, a.inP, BLK_B | BLK_C, y, dA, dC);
    const double r = y[3] - __ldg(a.aux + o);
    a.out[o] = ((i + j + k) & 1) == 0 ? r / dC : r;
  } else {
    const double T = __ldg(a.inP + o);
    double d = T;
    if ((i + j + k) & 1) {
      row_list<FORM, true>(g, i, j, k, a.inU, a.inP, BLK_C, y, dA, dC);
      d = (T + y[3]) / dC;
    }
    a.out[o] += a.omega * d;
  }
}

// ---- list rows by explicit stencils: 16 lanes per row ------------------------------
// The Gamma rows of a tiled level carry their explicit 4x4-block stencils
// (k_assemble_explicit, "explicit interface stencils").  Lane q < 15 of a
// row's 16-lane group takes Kuhn offset q: it loads the neighbour's 4 fields (masked:
// velocity 0 at Dirichlet / outside, pressure 0 outside -- level-0 inputs are the
// caller's vectors) and its 16 stencil entries, forms its part of the 4 row outputs;
// a 16-lane xor reduction sums them and lane 0 writes (same results as list_row).
constexpr int LX_NT = 128;
template <int FORM, int OP>
__global__ void __launch_bounds__(LX_NT) k_listx(DGrid g, StreamArgs a, const double* __restrict__ S0) {
  const int gt = blockIdx.x * LX_NT + threadIdx.x;
  const int e = gt >> 4, q = gt & 15;
  if (e >= a.nlist) return;  // whole 16-lane groups retire together
  const int t = __ldg(a.list + e);
  const int nx = g.n + 1;
  const int k = g.z0 + t / (nx * nx);
  const int rr = t % (nx * nx);
  const int i = rr % nx, j = rr / nx;
  const int64_t o = vidx(g, i, j, k);
  const unsigned em = elim(g, i, j, k);
  const double* S = S0 + (int64_t)e * EXPL;
  // which rows / columns this OP needs
  constexpr bool VROWS = OP == OP_APPLY || OP == OP_RESID || OP == OP_VEL;
  constexpr bool PROW = OP != OP_VEL;
  constexpr bool UCOL = OP != OP_P2;
  const bool c0 = ((i + j + k) & 1) == 0;  // pressure colour 0
  bool act = true;
  if (OP == OP_VEL) act = ((i + j + k) & (a.ncolors - 1)) == a.color && em != 7u;
  if (OP == OP_P2) act = !c0;
  double py[4] = {0.0, 0.0, 0.0, 0.0};
  // lanes of out-of-cube neighbours contribute 0 (their inputs are 0): they skip the
  // stencil loads, as do the rows of eliminated components (zero rows) -- boundary rows
  // of the free-slip / Dirichlet faces read a quarter to a half fewer stencil bytes
  const int dx = q < NQ ? kq_dx(q) : 0, dy = q < NQ ? kq_dy(q) : 0, dz = q < NQ ? kq_dz(q) : 0;
  const int xi = i + dx, yj = j + dy, zk = k + dz;
  const bool in = xi >= 0 && yj >= 0 && zk >= 0 && xi <= g.n && yj <= g.n && zk <= g.n;
  if (act && q < NQ && in) {
    const int n = g.n;
    const int64_t oc = o + dx + dy * g.px + dz * g.py;
    double u[3] = {0.0, 0.0, 0.0}, p = 0.0;
    if (UCOL) {
      const unsigned emv = in ? elim_mask(g.dirmask, g.slipmask, n, xi, yj, zk) : 7u;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double v = __ldg(a.inU + c * g.fs + oc);
        u[c] = ((emv >> c) & 1u) ? 0.0 : v;
      }
    }
    {
      const double v = __ldg(a.inP + oc);
      // P2: the masked T of R11 -- colour-0 neighbours only (odd offset sums)
      p = (in && (OP != OP_P2 || ((dx + dy + dz) & 1))) ? v : 0.0;
    }
    if (VROWS) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if ((em >> r) & 1u) continue;  // eliminated component: zero row
        const double2 s01 = __ldg(reinterpret_cast<const double2*>(S + (r * NQ + q) * 4));
        const double2 s23 = __ldg(reinterpret_cast<const double2*>(S + (r * NQ + q) * 4 + 2));
        const bool wA = OP == OP_VEL || OP == OP_RESID || (a.blocks & BLK_A);
        const bool wT = OP == OP_VEL || OP == OP_RESID || (a.blocks & BLK_BT);
        double v = 0.0;
        if (wA) v = fma(s01.x, u[0], fma(s01.y, u[1], s23.x * u[2]));
        if (wT) v = fma(s23.y, p, v);
        py[r] = v;
      }
    }
    if (PROW) {
      const double2 s23 = __ldg(reinterpret_cast<const double2*>(S + (3 * NQ + q) * 4 + 2));
      const bool wB = OP == OP_RESID || OP == OP_P1 || (OP == OP_APPLY && (a.blocks & BLK_B));
      const bool wC = OP != OP_APPLY || (a.blocks & BLK_C);
      double v = 0.0;
      if (wB && UCOL) {
        const double2 s01 = __ldg(reinterpret_cast<const double2*>(S + (3 * NQ + q) * 4));
        v = fma(s01.x, u[0], fma(s01.y, u[1], s23.x * u[2]));
      }
      if (wC) v = fma(s23.y, p, v);
      py[3] = v;
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if ((r < 3 && VROWS) || (r == 3 && PROW))
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) py[r] += __shfl_xor_sync(0xffffffffu, py[r], off);
  if (q != 0) return;
  const double* inv = S + 4 * NQ * 4;  // 1/A_00, 1/A_11, 1/A_22, 1/C
  if (OP == OP_APPLY || OP == OP_RESID) {
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      double v = ((em >> f) & 1u) ? 0.0 : py[f];
      if (OP == OP_RESID) v = ((em >> f) & 1u) ? 0.0 : __ldg(a.aux + f * g.fs + o) - py[f];
      a.out[f * g.fs + o] = v;
    }
  } else if (OP == OP_VEL) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const bool ec = (em >> c) & 1u;
      const double uc = ec ? 0.0 : __ldg(a.inU + c * g.fs + o);
      const double v = (act && !ec) ? fma(__ldg(a.aux + c * g.fs + o) - py[c], __ldg(inv + c), uc) : uc;
      if (a.cbuf) a.cbuf[(int64_t)e * 3 + c] = v;
      else a.out[c * g.fs + o] = v;
    }
  } else if (OP == OP_P1) {
    const double r = py[3] - __ldg(a.aux + o);
    a.out[o] = c0 ? r * __ldg(inv + 3) : r;
  } else {
    const double T = __ldg(a.inP + o);
    const double d = c0 ? T : (T + py[3]) * __ldg(inv + 3);
    a.out[o] += a.omega * d;
  }
}

constexpr int LIST_NT = 128;
template <int FORM, int OP>
__global__ void __launch_bounds__(LIST_NT) k_list(DGrid g, StreamArgs a) {
  const int e = blockIdx.x * LIST_NT + threadIdx.x;
  if (e >= a.nlist) return;
  const int t = a.list[e];
  const int nx = g.n + 1;
  const int k = g.z0 + t / (nx * nx);
  const int r = t % (nx * nx);
  list_row<FORM, OP>(g, a, r % nx, r / nx, k);
}

// ---- traction top-face rows (z = 1, isoviscous star): truncated stencils ----------
template <int FORM, int OP, int DX, int DY, int DZ>
__device__ __forceinline__ void top_off(Acc& acc, const double* const pls[3], int base) {
  if constexpr (kuhn(DX, DY, DZ) && DZ <= 0) {
    constexpr int NF = OP == OP_P2 ? 1 : 4;
    const double* q = pls[DZ + 1] + base + DY * HX + DX;
    if constexpr (OP == OP_P2) {
      constexpr double kC = KT<3, 0, 0, 0, DX, DY, DZ>::v;
      if constexpr (kC != 0.0) acc.C = fma(kC, q[0], acc.C);
    } else {
      const double u[3] = {q[0], q[FST], q[2 * FST]};
      const double p = q[3 * FST];
      (void)NF;
      if constexpr (OP != OP_P1) {
#define STK_TOP_A(a_, b_)                                                     \
  {                                                                           \
    constexpr double kA = KT<0, FORM, a_, b_, DX, DY, DZ>::v;                 \
    if constexpr (kA != 0.0) acc.A[a_] = fma(kA, u[b_], acc.A[a_]);           \
  }
        STK_TOP_A(0, 0) STK_TOP_A(0, 1) STK_TOP_A(0, 2)
        STK_TOP_A(1, 0) STK_TOP_A(1, 1) STK_TOP_A(1, 2)
        STK_TOP_A(2, 0) STK_TOP_A(2, 1) STK_TOP_A(2, 2)
#undef STK_TOP_A
        constexpr double kT0 = KT<1, 0, 0, 0, DX, DY, DZ>::v, kT1 = KT<1, 0, 1, 0, DX, DY, DZ>::v,
                         kT2 = KT<1, 0, 2, 0, DX, DY, DZ>::v;
        if constexpr (kT0 != 0.0) acc.BT[0] = fma(kT0, p, acc.BT[0]);
        if constexpr (kT1 != 0.0) acc.BT[1] = fma(kT1, p, acc.BT[1]);
        if constexpr (kT2 != 0.0) acc.BT[2] = fma(kT2, p, acc.BT[2]);
      }
      if constexpr (OP != OP_VEL) {
        constexpr double kB0 = KT<2, 0, 0, 0, DX, DY, DZ>::v, kB1 = KT<2, 0, 0, 1, DX, DY, DZ>::v,
                         kB2 = KT<2, 0, 0, 2, DX, DY, DZ>::v, kC = KT<3, 0, 0, 0, DX, DY, DZ>::v;
        if constexpr (kB0 != 0.0) acc.B = fma(kB0, u[0], acc.B);
        if constexpr (kB1 != 0.0) acc.B = fma(kB1, u[1], acc.B);
        if constexpr (kB2 != 0.0) acc.B = fma(kB2, u[2], acc.B);
        if constexpr (kC != 0.0) acc.C = fma(kC, p, acc.C);
      }
    }
  }
}
template <int FORM, int OP, int DZ>
__device__ __forceinline__ void top_plane(Acc& acc, const double* const pls[3], int base) {
  top_off<FORM, OP, -1, -1, DZ>(acc, pls, base);
  top_off<FORM, OP, 0, -1, DZ>(acc, pls, base);
  top_off<FORM, OP, 1, -1, DZ>(acc, pls, base);
  top_off<FORM, OP, -1, 0, DZ>(acc, pls, base);
  top_off<FORM, OP, 0, 0, DZ>(acc, pls, base);
  top_off<FORM, OP, 1, 0, DZ>(acc, pls, base);
  top_off<FORM, OP, -1, 1, DZ>(acc, pls, base);
  top_off<FORM, OP, 0, 1, DZ>(acc, pls, base);
  top_off<FORM, OP, 1, 1, DZ>(acc, pls, base);
}
// row of an isoviscous traction top-face vertex (code = CODE_TOP | class),
// from the staged planes k-1 (pls[0]) and k (pls[1])
template <int FORM, int OP>
__device__ __forceinline__ void finish_top(const DGrid& g, const StreamArgs& a, int i, int j, int k, int64_t o,
                                        uint8_t code, const double aux[4], const double* const pls[3], int base,
                                        const double* mt) {
  Acc acc;
  acc.zero();
  top_plane<FORM, OP, -1>(acc, pls, base);
  top_plane<FORM, OP, 0>(acc, pls, base);
  const int cl = code & (CODE_TOP - 1);
  const double h = g.h, mu = tab_ld(mt, cl), imu = tab_ld(mt, 256 + cl);
  const double sA = mu * h * (1.0 / 6.0), sB = h * h * (1.0 / 24.0), sC = g.delta * h * h * h * imu * (1.0 / 6.0);
  constexpr double kAd0 = KT<0, FORM, 0, 0, 0, 0, 0>::v, kAd1 = KT<0, FORM, 1, 1, 0, 0, 0>::v,
                   kAd2 = KT<0, FORM, 2, 2, 0, 0, 0>::v, kCd = KT<3, 0, 0, 0, 0, 0, 0>::v;
  if (OP == OP_APPLY || OP == OP_RESID) {
    const unsigned blk = OP == OP_APPLY ? a.blocks : BLK_ALL;
    double y[4];
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c] = ((blk & BLK_A) ? sA * acc.A[c] : 0.0) + ((blk & BLK_BT) ? sB * acc.BT[c] : 0.0);
    y[3] = ((blk & BLK_B) ? sB * acc.B : 0.0) - ((blk & BLK_C) ? sC * acc.C : 0.0);
#pragma unroll
    for (int f = 0; f < 4; ++f) a.out[f * g.fs + o] = OP == OP_RESID ? aux[f] - y[f] : y[f];
  } else if (OP == OP_VEL) {
    const bool act = ((i + j + k) & (a.ncolors - 1)) == a.color;
    const double isA = imu * (double)g.n * 6.0;
    const double ikd[3] = {1.0 / kAd0, 1.0 / kAd1, 1.0 / kAd2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double uc = pls[1][c * FST + base];
      a.out[c * g.fs + o] = act ? fma(aux[c] - fma(sA, acc.A[c], sB * acc.BT[c]), isA * ikd[c], uc) : uc;
    }
  } else if (OP == OP_P1) {
    const double r = fma(sB, acc.B, -sC * acc.C) - aux[3];
    a.out[o] = ((i + j + k) & 1) == 0 ? r * (mu * (6.0 / kCd) * g.idh3) : r;
  } else {
    const double T = pls[1][base];
    double d = T;
    if ((i + j + k) & 1) d = (T - sC * (acc.C - kCd * T)) * (mu * (6.0 / kCd) * g.idh3);
    a.out[o] = aux[3] + a.omega * d;
  }
}

// ---- stream role ----------------------------------------------------------------

// finishes output row k of this thread's column from the completed accumulator
template <int FORM, int OP>
__device__ __forceinline__ void finish_row(const DGrid& g, const StreamArgs& a, int i, int j, int k, int64_t o,
                                           uint8_t code, const double aux[4], const Acc& acc,
                                           const double* const pls[3], int base, const double* mt) {
  const double h = g.h;
  if (!(i > 0 && j > 0 && k > 0 && k < g.n)) {
    finish_boundary<OP>(g, a, i, j, k, code, acc.B, pls, base, mt);
    return;
  }
  const double mu = tab_ld(mt, code), imu = tab_ld(mt, 256 + code);
  const double sA = mu * h * (1.0 / 6.0);                       // 6A units
  const double sB = h * h * (1.0 / 24.0);                       // 24B, 24B^T units
  const double sC = g.delta * h * h * h * imu * (1.0 / 6.0);    // 6C units
  constexpr double kAd0 = KS<0, FORM, 0, 0, 0, 0, 0>::v, kAd1 = KS<0, FORM, 1, 1, 0, 0, 0>::v,
                   kAd2 = KS<0, FORM, 2, 2, 0, 0, 0>::v, kCd = KS<3, 0, 0, 0, 0, 0, 0>::v;
  if (OP == OP_APPLY || OP == OP_RESID) {
    double y[4];
    if (OP == OP_RESID || a.blocks == BLK_ALL) {
#pragma unroll
      for (int c = 0; c < 3; ++c) y[c] = fma(sA, acc.A[c], sB * acc.BT[c]);
      y[3] = fma(sB, acc.B, -sC * acc.C);
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        y[c] = ((a.blocks & BLK_A) ? sA * acc.A[c] : 0.0) + ((a.blocks & BLK_BT) ? sB * acc.BT[c] : 0.0);
      y[3] = ((a.blocks & BLK_B) ? sB * acc.B : 0.0) - ((a.blocks & BLK_C) ? sC * acc.C : 0.0);
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) a.out[f * g.fs + o] = OP == OP_RESID ? aux[f] - y[f] : y[f];
  } else if (OP == OP_VEL) {
    const bool act = ((i + j + k) & (a.ncolors - 1)) == a.color;
    const double* cpl = pls[1];
    // 1 / (sA kd) = 6 n / (mu kd): the Gauss-Seidel diagonal without a division
    const double isA = imu * (double)g.n * 6.0;
    const double ikd[3] = {1.0 / kAd0, 1.0 / kAd1, 1.0 / kAd2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double uc = cpl[c * FST + base];
      double v = uc;
      if (act) v = fma(aux[c] - fma(sA, acc.A[c], sB * acc.BT[c]), isA * ikd[c], uc);
      if (act || !a.inplace) a.out[c * g.fs + o] = v;
    }
  } else if (OP == OP_P1) {
    const double r = fma(sB, acc.B, -sC * acc.C) - aux[3];
    a.out[o] = ((i + j + k) & 1) == 0 ? r * (mu * (6.0 / kCd) * g.idh3) : r;
  } else {  // P2: acc.C = sum_o 6C(o) T (incl. the centre); neighbours of colour 1 are colour 0
    const double T = pls[1][base];
    double d = T;
    if ((i + j + k) & 1) d = (T - sC * (acc.C - kCd * T)) * (mu * (6.0 / kCd) * g.idh3);
    a.out[o] = aux[3] + a.omega * d;
  }
}

template <int FORM, int OP>
// register budget: 2 (apply / residual / velocity) or 3 (pressure passes) CTAs per SM
// with a little left over, so that one k_listx CTA (128 threads x 32 registers) can
// run next to the persistent stream CTAs and the Gamma rows overlap the stream
// (the residual spills at 120 and keeps 128: measured)
#ifndef STK_REGS_AR
#define STK_REGS_AR 120
#endif
#ifndef STK_REGS_P
#define STK_REGS_P 80
#endif
__global__ void __maxnreg__(OP == OP_RESID ? 128 : (OP == OP_APPLY || OP == OP_VEL) ? STK_REGS_AR : STK_REGS_P)
    k_stream(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapP,
             DGrid g,
             StreamArgs a) {
  constexpr int NF = OP == OP_P2 ? 1 : 4;
  constexpr int NA = n_aux(OP);
  constexpr int SLOT = slot_doubles(OP);
  constexpr uint32_t TX_BYTES = NF * PLANE * sizeof(double);
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem_raw =
      smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);  // 1 KB aligned TMA destinations
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + RING * SLOT * sizeof(double));
  double* auxb = reinterpret_cast<double*>(bars + RING);  // [2][NA][NT] per-thread aux double buffer

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int ntx = g.n / TX;
  const int tiles = ntx * (g.n / TY);
  const int nchunks = (g.nzl + a.kchunk - 1) / a.kchunk;
  const int nitems = tiles * nchunks;  // (tile, z-chunk), chunk-major: neighbours share L2
  const int G = gridDim.x;
  // geometry of item `it`: tile origin, output planes [kb, ke), planes kb-1..ke staged
  auto item_geom = [&](int it, int& ti0, int& tj0, int& tkb, int& tM) {
    const int tile = it % tiles, chunk = it / tiles;
    ti0 = (tile % ntx) * TX;
    tj0 = (tile / ntx) * TY;
    tkb = g.z0 + chunk * a.kchunk;
    tM = min(tkb + a.kchunk, g.z0 + g.nzl) - tkb + 2;
  };

#if STK_MU_SMEM
  __shared__ double s_mt[512];  // per-class mu [0..255] and 1/mu [256..511]
  for (int c = threadIdx.x; c < 512; c += NT) s_mt[c] = __ldg(g.mu + c);
  const double* mt = s_mt;
#else
  const double* mt = g.mu;
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#if STK_TMA_PREFETCH
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapU) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapP) : "memory");
#endif
  }
  __syncthreads();
  // Producer (thread 0): the planes of this CTA's items, items blockIdx.x + q G,
  // back to back; global plane sequence number S selects slot S % RING.
  int pq = 0, pp = 0, pS = 0, pi0 = 0, pj0 = 0, pkb = 0, pM = 0;
  bool pvalid = false;
  if (threadIdx.x == 0 && (int)blockIdx.x < nitems) {
    item_geom(blockIdx.x, pi0, pj0, pkb, pM);
    pvalid = true;
  }
  auto issue_next = [&]() {  // thread 0: stage the next plane of the sequence
    if (!pvalid) return;
    const int s = pS % RING;
    const int P = pkb - 1 + pp;
#if STK_TMA_FENCE
    fence_proxy_async();
#endif
    mbar_expect_tx(&bars[s], TX_BYTES);
    double* dst = ring + s * SLOT;
    if (NF == 4) {
      for (int f = 0; f < 3; ++f)
        tma_load_4d(dst + f * FST, &mapU, &bars[s], pi0 - 1 - a.ux0, pj0 - 1 - a.uy0, P - a.uz0, f);
      tma_load_4d(dst + 3 * FST, &mapP, &bars[s], pi0, pj0, P - g.z0 + 1, 0);
    } else {
      tma_load_4d(dst, &mapP, &bars[s], pi0, pj0, P - g.z0 + 1, 0);
    }
    ++pS;
    if (++pp == pM) {
      pp = 0;
      ++pq;
      const int it = blockIdx.x + pq * G;
      pvalid = it < nitems;
      if (pvalid) item_geom(it, pi0, pj0, pkb, pM);
    }
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < RING - 2; ++q) issue_next();  // consumer iteration S stages plane S+RING-2

  int S = 0;  // consumer: global plane sequence number
  // debug trace (a.trace != nullptr): cycles in the plane waits, the per-plane
  // barrier and the producer's issue, for thread 0 and for the last warp's lane 0
  const bool trc = a.trace != nullptr && (threadIdx.x == 0 || threadIdx.x == NT - 32);
  unsigned long long tw = 0, ts = 0, ti = 0, t_start = trc ? clock64() : 0;
  auto wait_plane = [&]() -> const double* {
    const int s = S % RING;
    const unsigned long long c0 = trc ? clock64() : 0;
    mbar_wait(&bars[s], (S / RING) & 1);
    if (trc) tw += clock64() - c0;
    return ring + s * SLOT;
  };
  auto release = [&]() {  // all reads of plane S-2 are done: stage a new plane into its slot
    const unsigned long long c0 = trc ? clock64() : 0;
    __syncthreads();
    const unsigned long long c1 = trc ? clock64() : 0;
    if (threadIdx.x == 0) issue_next();
    if (trc) {
      ts += c1 - c0;
      ti += clock64() - c1;
    }
    ++S;
  };
  const int i_ofs = tx, j_ofs = ty;
  const int base = (ty + 1) * HX + (tx + 1);

  for (int it = blockIdx.x; it < nitems; it += G) {
    int i0, j0, kb, M;
    item_geom(it, i0, j0, kb, M);
    const int kb1 = kb - 1;
    const bool last_x = i0 + TX == g.n, last_y = j0 + TY == g.n;
    const int i = i0 + i_ofs, j = j0 + j_ofs;
    // extra face rows: (n, j) for the last lane of last-x tiles, (i, n) for the
    // last warp of last-y tiles, (n, n) for the last thread of the corner tile
    const bool ex_x = last_x && tx == TX - 1, ex_y = last_y && ty == TY - 1, ex_c = ex_x && ex_y;
    const bool any_ex = last_x || last_y;

    // iteration m (plane P = kb-1+m) uses accumulators (acc0, acc1, acc2) for
    // outputs (P-1, P, P+1); R[] rotates by one per iteration (unrolled by 3)
    Acc R0, R1, R2;
    // m = 0 (plane kb-1): only output kb (its z-1 plane)
    R2.zero();
    accumulate<FORM, OP, -1>(R2, wait_plane(), base);
    release();
    // m = 1 (plane kb): outputs kb (in-plane) and kb+1 (z-1 plane)
    R0.zero();
    {
      const double* pl = wait_plane();
      accumulate3<FORM, OP, 6>(R0, R2, R0, pl, base);  // R2: in-plane (output kb), R0: output kb+1
    }
    release();
    int64_t o = vidx(g, i, j, kb);  // output row of the current iteration
    uint8_t code_nx = __ldg(g.code + o);
    // aux of row kb into buffer ab (cp.async group); each body prefetches the next row
    const double* auxsrc = OP == OP_P2 ? a.out : a.aux;
    auto aux_issue = [&](int64_t orow, int buf) {
#pragma unroll
      for (int f = 0; f < NA; ++f) cp_async8(auxb + (buf * NA + f) * NT + threadIdx.x, auxsrc + f * g.fs + orow);
      cp_async_commit();
    };
    int ab = 0;
    if (NA > 0) aux_issue(o, ab);

    auto body = [&](int m, Acc& acc0, Acc& acc1, Acc& acc2) {
      const int k = kb1 + m - 1;  // output finished in this iteration
      acc2.zero();
      // per-output data of row k, staged with plane k (previous slot, landed)
      const uint8_t code = code_nx;           // loaded one iteration ahead
      code_nx = __ldg(g.code + o + g.py);     // next row (the code array holds the halo planes)
      uint8_t cxy[3] = {0xFF, 0xFF, 0xFF};
      if (any_ex) {
        if (ex_x) cxy[0] = __ldg(g.code + o + 1);
        if (ex_y) cxy[1] = __ldg(g.code + o + g.px);
        if (ex_c) cxy[2] = __ldg(g.code + o + g.px + 1);
      }
      double aux[4] = {0, 0, 0, 0};
      if (NA > 0) {
        aux_issue(o + g.py, ab ^ 1);  // next row (the slab holds the halo planes)
        cp_async_wait1();             // this row's group has landed
#pragma unroll
        for (int f = 0; f < NA; ++f) aux[OP == OP_RESID || OP == OP_VEL ? f : 3] = auxb[(ab * NA + f) * NT + threadIdx.x];
        ab ^= 1;
      }
      const double* pl = wait_plane();
      // plane P is output P-1's z+1 plane, output P's own plane, output P+1's z-1 plane
      if (m < M - 1) accumulate3<FORM, OP, 7>(acc0, acc1, acc2, pl, base);
      else accumulate3<FORM, OP, 1>(acc0, acc1, acc2, pl, base);
      const double* pls[3] = {ring + ((S + RING - 2) % RING) * SLOT, ring + ((S + RING - 1) % RING) * SLOT, pl};
      if (!(code & (0x80 | CODE_TOP))) {
        finish_row<FORM, OP>(g, a, i, j, k, o, code, aux, acc0, pls, base, mt);
      } else if (code != CODE_IRREGULAR && !(OP == OP_VEL && a.inplace)) {
        finish_top<FORM, OP>(g, a, i, j, k, o, code, aux, pls, base, mt);
      }
      // face rows i = n, j = n (Dirichlet with an isoviscous star, else list rows)
      if (any_ex) {
        if (ex_x && !(cxy[0] & 0x80)) {
          const double Bu = (OP == OP_P2 || OP == OP_VEL) ? 0.0 : b_row_smem<true, false>(pls, base + 1);
          finish_boundary<OP>(g, a, g.n, j, k, cxy[0], Bu, pls, base + 1, mt);
        }
        if (ex_y && !(cxy[1] & 0x80)) {
          const double Bu = (OP == OP_P2 || OP == OP_VEL) ? 0.0 : b_row_smem<false, true>(pls, base + HX);
          finish_boundary<OP>(g, a, i, g.n, k, cxy[1], Bu, pls, base + HX, mt);
        }
        if (ex_c && !(cxy[2] & 0x80)) {
          const double Bu = (OP == OP_P2 || OP == OP_VEL) ? 0.0 : b_row_smem<true, true>(pls, base + HX + 1);
          finish_boundary<OP>(g, a, g.n, g.n, k, cxy[2], Bu, pls, base + HX + 1, mt);
        }
      }
      release();
      o += g.py;
    };
#ifndef STK_UNROLL3_MASK
#define STK_UNROLL3_MASK (1 << OP_VEL)
#endif
    if constexpr (!((STK_UNROLL3_MASK >> OP) & 1)) {
      // one body instance, the accumulators rotate by register moves: 3x less code
      // (measured faster for these OPs; the velocity pass keeps the 3-way unroll)
#pragma unroll 1
      for (int m = 2; m < M; ++m) {
        body(m, R2, R0, R1);
        R2 = R0;
        R0 = R1;
      }
    } else {
      int m = 2;
      for (; m + 2 < M; m += 3) {
        body(m, R2, R0, R1);
        body(m + 1, R0, R1, R2);
        body(m + 2, R1, R2, R0);
      }
      if (m < M) body(m, R2, R0, R1);
      if (m + 1 < M) body(m + 1, R0, R1, R2);
    }
  }
  if (trc) {
    unsigned long long* d = a.trace + (blockIdx.x * 2 + (threadIdx.x ? 1 : 0)) * 5;
    d[0] = clock64() - t_start;
    d[1] = tw;
    d[2] = ts;
    d[3] = ti;
    d[4] = S;
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
                     int y1, int z0v, int z1v, unsigned bx = HX, unsigned by = HY) {
  PFN_encodeTiled enc = encoder();
  if (!enc) return false;
  const double* origin = base + vidx_host(g, x0, y0, z0v);
  cuuint64_t dims[4] = {(cuuint64_t)(x1 - x0 + 1), (cuuint64_t)(y1 - y0 + 1), (cuuint64_t)(z1v - z0v + 1),
                        (cuuint64_t)nfields};
  cuuint64_t strides[3] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.py * 8, (cuuint64_t)g.fs * 8};
  cuuint32_t box[4] = {bx, by, 1, 1};
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
  // the assembled stencils must equal the compile-time integer stencils the kernels use
  std::vector<double> hst(cnt);
  ok &= cudaMemcpyAsync(hst.data(), d, cnt * sizeof(double), cudaMemcpyDeviceToHost, st) == cudaSuccess;
  ok &= cudaStreamSynchronize(st) == cudaSuccess;
  for (int o = 0; ok && o < 27; ++o) {
    const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
    for (int f = 0; f < 3; ++f)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          ok &= std::fabs(hst[((f * 3 + a) * 3 + b) * 27 + o] - kst(0, f, a, b, dx, dy, dz) / 6.0) <= 1e-14;
    for (int a = 0; a < 3; ++a) {
      ok &= std::fabs(hst[729 + a * 27 + o] - kst(1, 0, a, 0, dx, dy, dz) / 24.0) <= 1e-14;
      ok &= std::fabs(hst[810 + a * 27 + o] - kst(2, 0, 0, a, dx, dy, dz) / 24.0) <= 1e-14;
    }
    ok &= std::fabs(hst[891 + o] - kst(3, 0, 0, 0, dx, dy, dz) / 6.0) <= 1e-14;
  }
  cudaFree(d);
  done = ok;
  return ok;
}

inline size_t stream_smem(int op) {
  return 1024 + RING * slot_doubles(op) * sizeof(double) + RING * sizeof(uint64_t) + 2 * n_aux(op) * NT * sizeof(double);
}

// the irregular-row list of a level (built by stk_assemble)
struct ListView {
  const int32_t* list;
  int n;
  const double* S;                // explicit stencils of the list rows [n][EXPL] (nullptr: element loop)
  cudaStream_t side;              // list kernel runs here, concurrently (nullptr: same stream)
  cudaEvent_t ev_fork, ev_join;
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
  // persistent grid: every resident CTA slot, items (tile, z-chunk) round robin
  static const int kchunk_env = getenv("STK_KCHUNK") ? atoi(getenv("STK_KCHUNK")) : 0;
  static int slots = 0;
  if (!slots) {
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stream<FORM, OP>, NT, sm);
    slots = std::max(1, nsm * std::max(1, per_sm));
  }
  // chunk length: >= ~4 items per CTA for balance, 4..16 planes (short chunks keep
  // concurrently streaming neighbour tiles at the same height: halos shared in L2)
  // (measured, profiles/r02_stream_kchunk_sweep.log: 16 planes is within 1 % of the best at
  // n = 256; 32 planes win 3 % per kernel at n = 512 but are not adopted, see DESIGN 8)
  const int want = std::max(1, (4 * slots + tiles - 1) / tiles);
  int kc = kchunk_env > 0 ? kchunk_env : std::min(16, std::max(4, (g.nzl + want - 1) / want));
  kc = std::max(1, std::min(kc, g.nzl));
  const int chunks = (g.nzl + kc - 1) / kc;
  const int nitems = tiles * chunks;
  const int grid = std::min(nitems, slots);
  a.kchunk = kc;
  a.inU = inU;
  a.inP = inP;
  a.list = lv.list;
  a.nlist = lv.n;
  static const int fork_env = getenv("STK_LIST_FORK") ? atoi(getenv("STK_LIST_FORK")) : 1;
  const bool do_list = lv.n > 0;
  // In-place velocity pass: the list rows (into cbuf) must read start-of-pass values; the
  // face rows with truncated stencils (free slip, traction) couple to same-colour regular
  // rows, which the stream kernel relaxes in place -- so the list kernel runs first, on
  // the same stream (no overlap, deterministic).
  // (Dirichlet-only levels have no such rows -- Gamma_12 rows couple to other-colour or
  // Gamma columns only -- and keep the overlapped fork.)
  const bool face_rows = g.slipmask != 0u || (g.dirmask & 63u) != 63u;
  const bool list_first = do_list && OP == OP_VEL && a.inplace && lv.S != nullptr && face_rows;
  const bool fork = do_list && !list_first && fork_env && lv.side != nullptr;
  if (fork) {
    if (cudaEventRecord(lv.ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(lv.side, lv.ev_fork, 0) != cudaSuccess)
      return false;
  }
  static const bool trace = getenv("STK_STREAM_TRACE") && atoi(getenv("STK_STREAM_TRACE"));
  static unsigned long long* tbuf = nullptr;
  if (trace && !tbuf) cudaMallocManaged(&tbuf, sizeof(unsigned long long) * 4096 * 10);
  a.trace = trace ? tbuf : nullptr;
  if (list_first)
    k_listx<FORM, OP><<<(unsigned)(((int64_t)lv.n * 16 + LX_NT - 1) / LX_NT), LX_NT, 0, st>>>(g, a, lv.S);
  k_stream<FORM, OP><<<dim3(grid), NT, sm, st>>>(mU, mP, g, a);
  if (trace) {  // debug: mean per-CTA cycle split of this launch
    cudaStreamSynchronize(st);
    double tot[2][5] = {};
    for (int b = 0; b < grid; ++b)
      for (int r = 0; r < 2; ++r)
        for (int q = 0; q < 5; ++q) tot[r][q] += (double)tbuf[(b * 2 + r) * 5 + q] / grid;
    fprintf(stderr, "k_stream<%d,%d> n=%d grid=%d kc=%d planes/CTA %.1f | thread0: total %.0f wait %.0f sync %.0f issue %.0f"
            " | last warp: total %.0f wait %.0f sync %.0f (cycles)\n", FORM, OP, g.n, grid, kc, tot[0][4], tot[0][0],
            tot[0][1], tot[0][2], tot[0][3], tot[1][0], tot[1][1], tot[1][2]);
  }
  if (do_list && !list_first) {
    if (lv.S) k_listx<FORM, OP><<<(unsigned)(((int64_t)lv.n * 16 + LX_NT - 1) / LX_NT), LX_NT, 0, fork ? lv.side : st>>>(g, a, lv.S);
    else k_list<FORM, OP><<<(lv.n + LIST_NT - 1) / LIST_NT, LIST_NT, 0, fork ? lv.side : st>>>(g, a);
  }
  if (fork) {
    if (cudaEventRecord(lv.ev_join, lv.side) != cudaSuccess || cudaStreamWaitEvent(st, lv.ev_join, 0) != cudaSuccess)
      return false;
  }
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
// The second pass of the middle colour pair of the symmetric sweep (colours
// 0..nc-1, nc-1..0; R12) repeats the relaxation of the same colour.  A regular row of
// the mod / grad forms couples only to other colours (7-point A) and to
// its own component (diagonal centre block), so the repeat reproduces it exactly in
// exact arithmetic (to rounding in fp64): only the rows that couple within the colour
// change -- the list rows (Gamma_12, Gamma_F) and the isoviscous traction-face rows
// (truncated stencils).  So: u_out = u_in (one device copy of the 3 velocity fields),
// then those rows are relaxed from u_in (k_listx over the "repeat list").  Same
// result as the full pass up to rounding.
template <int FORM>
bool launch_vel_repeat_t(const DGrid& g, const ListView& lv, const double* uin, const double* p, const double* b,
                         double* uout, int color, int ncolors, cudaStream_t st) {
  if (cudaMemcpyAsync(uout, uin, sizeof(double) * 3 * g.fs, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return false;
  if (lv.n == 0) return true;
  StreamArgs a{};
  a.out = uout;
  a.aux = b;
  a.color = color;
  a.ncolors = ncolors;
  a.inU = uin;
  a.inP = p;
  a.list = lv.list;
  a.nlist = lv.n;
  if (lv.S) k_listx<FORM, OP_VEL><<<(unsigned)(((int64_t)lv.n * 16 + LX_NT - 1) / LX_NT), LX_NT, 0, st>>>(g, a, lv.S);
  else k_list<FORM, OP_VEL><<<(lv.n + LIST_NT - 1) / LIST_NT, LIST_NT, 0, st>>>(g, a);
  return true;
}
inline bool launch_vel_repeat(int form, DGrid g, const ListView& lv, const double* uin, const double* p,
                              const double* b, double* uout, int color, int ncolors, cudaStream_t st) {
  switch (form) {
    case FORM_MOD: return launch_vel_repeat_t<FORM_MOD>(g, lv, uin, p, b, uout, color, ncolors, st);
    case FORM_SYM: return launch_vel_repeat_t<FORM_SYM>(g, lv, uin, p, b, uout, color, ncolors, st);
    default: return launch_vel_repeat_t<FORM_GRAD>(g, lv, uin, p, b, uout, color, ncolors, st);
  }
}
// list rows' results of an in-place velocity pass back into the vector
__global__ void k_scatter3(DGrid g, const int32_t* __restrict__ list, int n, const double* __restrict__ cbuf,
                           double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int t = __ldg(list + e);
  const int nx = g.n + 1;
  const int k = g.z0 + t / (nx * nx), rr = t % (nx * nx);
  const int64_t o = vidx(g, rr % nx, rr / nx, k);
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c * g.fs + o] = cbuf[(int64_t)e * 3 + c];
}
// In-place velocity colour pass (mod / grad forms): u is updated in place.  A regular
// row of the active colour couples only to the other colour (7-point A), so
// its in-place update reads exactly the start-of-pass values; the list rows (Gamma_12,
// Gamma_F, lv = the repeat list incl. the isoviscous traction-face rows) are computed
// from the start-of-pass vector into cbuf (their coefficients to same-colour regular
// neighbours are exactly 0) and scattered after the stream kernel.  No ping-pong copy.
// list_only: the repeat pass of the middle colour (regular rows unchanged, R12).
template <int FORM>
bool launch_vel_inplace_t(const DGrid& g, const ListView& lv, double* u, const double* p, const double* b,
                          double* cbuf, int color, int ncolors, bool list_only, cudaStream_t st) {
  StreamArgs a{};
  a.out = u;
  a.aux = b;
  a.color = color;
  a.ncolors = ncolors;
  a.inplace = 1;
  a.cbuf = cbuf;
  if (list_only) {
    if (lv.n == 0) return true;
    a.inU = u;
    a.inP = p;
    a.list = lv.list;
    a.nlist = lv.n;
    k_listx<FORM, OP_VEL><<<(unsigned)(((int64_t)lv.n * 16 + LX_NT - 1) / LX_NT), LX_NT, 0, st>>>(g, a, lv.S);
  } else if (!launch_stream_t<FORM, OP_VEL>(g, u, p, lv, a, st)) {
    return false;
  }
  if (lv.n > 0) k_scatter3<<<(lv.n + 255) / 256, 256, 0, st>>>(g, lv.list, lv.n, cbuf, u);
  return true;
}
inline bool launch_vel_inplace(int form, DGrid g, const ListView& lv, double* u, const double* p, const double* b,
                               double* cbuf, int color, int ncolors, bool list_only, cudaStream_t st) {
  if (!lv.S) return false;  // needs the explicit stencils of the list rows
  switch (form) {
    case FORM_MOD: return launch_vel_inplace_t<FORM_MOD>(g, lv, u, p, b, cbuf, color, ncolors, list_only, st);
    case FORM_GRAD: return launch_vel_inplace_t<FORM_GRAD>(g, lv, u, p, b, cbuf, color, ncolors, list_only, st);
    default: return false;  // sym: the centre block couples the components; ping-pong passes
  }
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
