// Tiled constant-stencil kernels for levels with n >= 64 (the hot path).
//
// Design:
//  * a CTA owns a TX x TY column tile of the slab and marches through a chunk of
//    z-planes; each plane of the 4 input fields (with a 1-vertex xy halo) is
//    staged in shared memory by ONE TMA box load (cp.async.bulk.tensor.4d,
//    mbarrier complete_tx), PREF planes ahead, in a ring of PREF+2 slots;
//  * plane-streaming accumulation: when plane P lands, every thread reads the 7
//    in-plane points of its column once and adds their contributions to the rows
//    of the three outputs (P-1, P, P+1) of its column (the 15-point Kuhn stencil
//    spans three planes), so each input value is read from shared memory once per
//    output row role and HBM traffic is one read of x + one write of y;
//  * regular rows (interior vertex, isoviscous 24-tet star: class k) use the
//    constant unit stencils assembled once by k_assemble_stencils,
//    scaled by mu_k h (A), h^2 (B, B^T) and delta h^3 / mu_k (C);
//  * irregular rows (Gamma_12, boundary / Gamma_F: P:355-360) of the finished
//    output plane are compacted in shared memory and evaluated by the element
//    loop row_generic reading the same staged planes (no extra HBM traffic).
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
  int kchunk;           // output planes per CTA
  unsigned blocks;      // APPLY block mask
  int color, ncolors;   // VEL
  double omega;         // P2
  int no_tma;           // debug: stage planes with plain loads instead of TMA
  int skip_irr;         // debug (timing only): skip the irregular rows
  const double* inA;    // (no_tma) base of the staged fields
  const double* inB;    // (no_tma, VEL) pressure field
};

// shared-memory fetch for row_generic: planes staged in the ring
template <int NF>
struct FetchSmem {
  const double* ring;
  int i0, j0, kb1;  // tile origin, plane of ring index 0 (kb - 1)
  bool red_only;    // P2: pressure = T at colour-0 vertices only, velocity 0
  __device__ __forceinline__ double operator()(const DGrid& g, int i, int j, int k, int f) const {
    const int slot = (k - kb1) % RING;
    const int li = i - i0 + 1, lj = j - j0 + 1;
    if (NF == 1) {
      if (f != 3 || (red_only && ((i + j + k) & 1))) return 0.0;
      return ring[slot * FST + lj * HX + li];
    }
    if (f < 3 && is_dirichlet(g, i, j, k)) return 0.0;
    return ring[(slot * NF + f) * FST + lj * HX + li];
  }
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
  constexpr int NF = OP == OP_P2 ? 1 : 4;
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
  (void)NF;
}

template <int FORM, int OP>
__global__ void __launch_bounds__(NT, 2)
    k_stream(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, DGrid g,
             StreamArgs a) {
  constexpr int NF = OP == OP_P2 ? 1 : 4;
  constexpr uint32_t SLOT_BYTES = NF * FST * sizeof(double);
  constexpr uint32_t TX_BYTES = NF * PLANE * sizeof(double);  // bytes landed per plane
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem_raw =
      smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);  // 1 KB aligned TMA destinations
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + RING * SLOT_BYTES);
  int* irr_cnt = reinterpret_cast<int*>(bars + RING);
  int* irr_list = irr_cnt + 1;

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int ntx = g.n / TX;
  const int i0 = (blockIdx.x % ntx) * TX, j0 = (blockIdx.x / ntx) * TY;
  const int kb = g.z0 + blockIdx.y * a.kchunk;
  const int ke = min(kb + a.kchunk, g.z0 + g.nzl);
  if (kb >= ke) return;
  const int M = ke - kb + 2;  // planes kb-1 .. ke
  const int kb1 = kb - 1;
  const bool last_x = i0 + TX == g.n, last_y = j0 + TY == g.n;
  const int i = i0 + tx, j = j0 + ty;
  const int base = (ty + 1) * HX + (tx + 1);
  const double h = g.h;
  const double sA = h, sB = h * h, sC = g.delta * h * h * h;  // times mu / 1 / 1/mu

  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&bars[s], 1);
    *irr_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto stage_plain = [&](int m) {  // debug path: cooperative plain loads, synchronous
    const int s = m % RING;
    const int zl = kb1 + m - g.z0 + 1;
    for (int e = threadIdx.x; e < NF * PLANE; e += NT) {
      const int f = e / PLANE, r = e % PLANE;
      const int li = r % HX, lj = r / HX;
      const int gi = i0 - 1 + li, gj = j0 - 1 + lj;
      double v = 0.0;
      if (gi >= 0 && gj >= 0 && gi <= g.n && gj <= g.n) {
        const double* src = (OP == OP_VEL && f == 3) ? a.inB : a.inA + (OP == OP_VEL ? f : f) * g.fs;
        v = src[(int64_t)zl * g.py + (int64_t)(gj + 1) * g.px + (gi + 1)];
      }
      ring[(s * NF + f) * FST + r] = v;
    }
  };
  auto issue = [&](int m) {
    if (a.no_tma) return;
    if (m >= M) return;
    const int s = m % RING;
    const int zc = kb1 + m - g.z0 + 1;  // local plane index of the layout
    fence_proxy_async();
    mbar_expect_tx(&bars[s], TX_BYTES);
    double* dst = ring + s * NF * FST;
    if (OP == OP_VEL) {
      // box origin (i0-1, j0-1) in vertex coordinates = (i0, j0) in the ghost-framed layout
      for (int f = 0; f < 3; ++f) tma_load_4d(dst + f * FST, &mapA, &bars[s], i0, j0, zc, f);  // u
      tma_load_4d(dst + 3 * FST, &mapB, &bars[s], i0, j0, zc, 0);                            // p
    } else {
      for (int f = 0; f < NF; ++f) tma_load_4d(dst + f * FST, &mapA, &bars[s], i0, j0, zc, f);
    }
  };
  if (threadIdx.x == 0)
    for (int m = 0; m < PREF; ++m) issue(m);

  Acc acc0, acc1, acc2;  // outputs P-1, P, P+1
  acc0.zero();
  acc1.zero();
  acc2.zero();
  const FetchSmem<NF> fsm{ring, i0, j0, kb1, OP == OP_P2};

  for (int m = 0; m < M; ++m) {
    const int P = kb1 + m;
    const int k = P - 1;  // output finished in this iteration
    // early loads of per-output data (code byte, own auxiliary values)
    uint8_t code = CODE_IRREGULAR;
    double aux[4] = {0, 0, 0, 0};
    double own_p = 0.0;
    const bool fin = m >= 2;
    if (fin) {
      const int64_t o = vidx(g, i, j, k);
      code = __ldg(g.code + o);
      if (OP == OP_RESID) {
#pragma unroll
        for (int f = 0; f < 4; ++f) aux[f] = __ldg(a.aux + f * g.fs + o);
      } else if (OP == OP_VEL) {
#pragma unroll
        for (int f = 0; f < 3; ++f) aux[f] = __ldg(a.aux + f * g.fs + o);
      } else if (OP == OP_P1) {
        aux[3] = __ldg(a.aux + o);
      } else if (OP == OP_P2) {
        own_p = a.out[o];
      }
    }
    const int s = m % RING;
    if (a.no_tma) {
      stage_plain(m);
      __syncthreads();
    } else {
      mbar_wait(&bars[s], (m / RING) & 1);
    }
    const double* pl = ring + s * NF * FST;
    // inputs at Dirichlet velocity DoFs are ignored: zero them in the staged plane
    if (NF == 4) {
      const unsigned dm = g.dirmask;
      const bool mplane = ((dm & 16u) && P == 0) || ((dm & 32u) && P == g.n);
      const bool mx0 = (dm & 1u) && i0 == 0, mx1 = (dm & 2u) && last_x;
      const bool my0 = (dm & 4u) && j0 == 0, my1 = (dm & 8u) && last_y;
      if (mplane || mx0 || mx1 || my0 || my1) {
        double* w = ring + s * NF * FST;
        for (int e = threadIdx.x; e < 3 * PLANE; e += NT) {
          const int f = e / PLANE, r = e % PLANE, li = r % HX, lj = r / HX;
          if (mplane || (mx0 && li == 1) || (mx1 && li == TX + 1) || (my0 && lj == 1) || (my1 && lj == TY + 1))
            w[f * FST + r] = 0.0;
        }
        __syncthreads();
      }
    }
    accumulate<FORM, OP, 1>(acc0, pl, base);   // plane P is output P-1's z+1 plane
    accumulate<FORM, OP, 0>(acc1, pl, base);
    accumulate<FORM, OP, -1>(acc2, pl, base);

    if (fin) {
      const int64_t o = vidx(g, i, j, k);
      const double* cpl = ring + ((m - 1) % RING) * NF * FST;  // plane k
      if (code != CODE_IRREGULAR) {
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
          const double T = cpl[base];
          double d = T;
          if ((i + j + k) & 1) {
            const double off = acc0.C - st_C[13] * T;  // neighbours only (all colour 0)
            d = (T - sC * imu * off) / (sC * imu * st_C[13]);
          }
          a.out[o] = own_p + a.omega * d;
        }
      } else {
        irr_list[atomicAdd(irr_cnt, 1)] = (ty + 1) * HX + (tx + 1);
      }
      // edge column i = n / row j = n of the last tiles: boundary rows
      if (last_x && tx == 0) irr_list[atomicAdd(irr_cnt, 1)] = (ty + 1) * HX + (TX + 1);
      if (last_y && ty == 0) irr_list[atomicAdd(irr_cnt, 1)] = (TY + 1) * HX + (tx + 1);
      if (last_x && last_y && threadIdx.x == 0) irr_list[atomicAdd(irr_cnt, 1)] = (TY + 1) * HX + (TX + 1);
    }
    __syncthreads();
    if (fin && !a.skip_irr) {
      const int cnt = *irr_cnt;
      for (int q = threadIdx.x; q < cnt; q += NT) {
        const int e = irr_list[q];
        const int ii = i0 + (e % HX) - 1, jj = j0 + (e / HX) - 1;
        const int64_t o = vidx(g, ii, jj, k);
        double y[4], dA[3], dC;
        const bool dir = is_dirichlet(g, ii, jj, k);
        if (OP == OP_APPLY || OP == OP_RESID) {
          row_generic<FORM>(g, ii, jj, k, fsm, OP == OP_APPLY ? a.blocks : BLK_ALL, y, dA, dC);
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            double v = y[f];
            if (OP == OP_RESID) v = (f < 3 && dir) ? 0.0 : __ldg(a.aux + f * g.fs + o) - y[f];
            a.out[f * g.fs + o] = v;
          }
        } else if (OP == OP_VEL) {
          const bool act = ((ii + jj + k) % a.ncolors) == a.color && !dir;
          if (act) row_generic<FORM>(g, ii, jj, k, fsm, BLK_A | BLK_BT, y, dA, dC);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double uc = dir ? 0.0 : ring[((m - 1) % RING * NF + c) * FST + e];
            a.out[c * g.fs + o] = act ? uc + (__ldg(a.aux + c * g.fs + o) - y[c]) / dA[c] : uc;
          }
        } else if (OP == OP_P1) {
          row_generic<FORM>(g, ii, jj, k, fsm, BLK_B | BLK_C, y, dA, dC);
          const double r = y[3] - __ldg(a.aux + o);
          a.out[o] = ((ii + jj + k) & 1) == 0 ? r / dC : r;
        } else {
          const double T = ring[((m - 1) % RING) * FST + e];
          double d = T;
          if ((ii + jj + k) & 1) {
            row_generic<FORM>(g, ii, jj, k, fsm, BLK_C, y, dA, dC);
            d = (T + y[3]) / dC;
          }
          a.out[o] += a.omega * d;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      *irr_cnt = 0;
      issue(m + PREF);
    }
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

inline bool make_map(CUtensorMap* map, const double* base, const DGrid& g, int box_fields) {
  PFN_encodeTiled enc = encoder();
  if (!enc) return false;
  // ghost-framed extent: positions 0..n+1 hold vertices -1..n (boxes never leave it)
  cuuint64_t dims[4] = {(cuuint64_t)(g.n + 2), (cuuint64_t)(g.n + 2), (cuuint64_t)(g.nzl + 2), (cuuint64_t)box_fields};
  cuuint64_t strides[3] = {(cuuint64_t)g.px * 8, (cuuint64_t)g.py * 8, (cuuint64_t)g.fs * 8};
  cuuint32_t box[4] = {HX, HY, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es,
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
  return 1024 + RING * NF * FST * sizeof(double) + RING * sizeof(uint64_t) + sizeof(int) * (1 + (TX + 1) * (TY + 1) + 8);
}

template <int FORM, int OP>
bool launch_stream_t(const DGrid& g, const double* inA, const double* inB, int nfA, const StreamArgs& a0,
                     cudaStream_t st) {
  CUtensorMap mA, mB;
  if (!make_map(&mA, inA, g, nfA)) return false;
  if (!make_map(&mB, inB ? inB : inA, g, 1)) return false;
  const size_t sm = stream_smem(OP);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_stream<FORM, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
      return false;
    attr = true;
  }
  const int tiles = (g.n / TX) * (g.n / TY);
  const int target = 148 * 2 * 6;
  int chunks = (target + tiles - 1) / tiles;
  chunks = std::max(1, std::min(chunks, g.nzl / 8));
  StreamArgs a = a0;
  static const int no_tma = getenv("STK_NO_TMA") ? atoi(getenv("STK_NO_TMA")) : 0;
  a.no_tma = no_tma;
  static const int skip_irr = getenv("STK_SKIP_IRR") ? atoi(getenv("STK_SKIP_IRR")) : 0;
  a.skip_irr = skip_irr;
  a.inA = inA;
  a.inB = inB;
  a.kchunk = (g.nzl + chunks - 1) / chunks;
  chunks = (g.nzl + a.kchunk - 1) / a.kchunk;
  k_stream<FORM, OP><<<dim3(tiles, chunks), NT, sm, st>>>(mA, mB, g, a);
  return true;
}

template <int OP>
bool launch_stream(int form, const DGrid& g, const double* inA, const double* inB, int nfA, const StreamArgs& a,
                   cudaStream_t st) {
  switch (form) {
    case FORM_MOD: return launch_stream_t<FORM_MOD, OP>(g, inA, inB, nfA, a, st);
    case FORM_SYM: return launch_stream_t<FORM_SYM, OP>(g, inA, inB, nfA, a, st);
    default: return launch_stream_t<FORM_GRAD, OP>(g, inA, inB, nfA, a, st);
  }
}

inline bool launch_apply_tiled(int form, DGrid g, const double* x, double* y, unsigned blocks, cudaStream_t st) {
  StreamArgs a{};
  a.out = y;
  a.blocks = blocks;
  return launch_stream<OP_APPLY>(form, g, x, nullptr, 4, a, st);
}
inline bool launch_residual_tiled(int form, DGrid g, const double* x, const double* b, double* r, cudaStream_t st) {
  StreamArgs a{};
  a.out = r;
  a.aux = b;
  a.blocks = BLK_ALL;
  return launch_stream<OP_RESID>(form, g, x, nullptr, 4, a, st);
}
inline bool launch_vel_pass_tiled(int form, DGrid g, const double* uin, const double* p, const double* b,
                                  double* uout, int color, int ncolors, cudaStream_t st) {
  StreamArgs a{};
  a.out = uout;
  a.aux = b;
  a.color = color;
  a.ncolors = ncolors;
  return launch_stream<OP_VEL>(form, g, uin, p, 3, a, st);
}
inline bool launch_p_pass1_tiled(int form, DGrid g, const double* x, const double* gp, double* T, cudaStream_t st) {
  StreamArgs a{};
  a.out = T;
  a.aux = gp;
  return launch_stream<OP_P1>(form, g, x, nullptr, 4, a, st);
}
inline bool launch_p_pass2_tiled(int form, DGrid g, const double* T, double* p, double omega, cudaStream_t st) {
  StreamArgs a{};
  a.out = p;
  a.omega = omega;
  return launch_stream<OP_P2>(form, g, T, nullptr, 1, a, st);
}

}  // namespace stk
