// Fused forward Gauss-Seidel sweep of the velocity smoother (colour 0, then colour 1)
// in ONE z-marching pass (mod / grad forms, red-black colours, tiled levels n >= 64).
//
// The symmetric sweep of Â (reading R12) is 0, 1, (1), 0.  A regular row of
// the mod / grad forms is the 7-point mu-Laplacian, so a colour-c row
// couples only to colour 1-c: the colour-1 pass needs the colour-0 values of the
// same sweep at the 6 axis neighbours, i.e. at planes k-1, k, k+1.  Marching in z, the
// kernel relaxes colour 0 on plane k+1 (R1, from the old colour-1 values) and then
// colour 1 on plane k (B, from the R1 values of planes k-1..k+1 and its own old
// value) -- one read of (u, p, f), one write of u: the 80 B two-colour sweep of
// SURVEY §8(d) instead of two 81 B passes.
//
//  * Tiles of 32 x 8 columns; the staged planes carry a 2-vertex xy ring (box 38 x 12
//    from vertex (i0 - 3, j0 - 2): TMA over the whole stored slab incl. its ghost frame;
//    the x start coordinate must be EVEN for fp64 -- a 16-byte aligned box row -- or the
//    copy raises an illegal instruction on sm_100a, tools/probe_tma_sweep.cu) because B
//    at a tile edge needs R1 at the neighbouring
//    column, which this CTA relaxes itself (ring 1, redundantly with the neighbouring
//    tile) from the old values of ring 2.  The velocity of Dirichlet-face vertices is
//    zeroed in shared memory after each plane lands (inputs there are ignored, API).
//    R1 results overwrite the red entries of the staged slot in place: later R1 steps
//    read only black values.
//  * A z-chunk [kb, ke) relaxes R1 on planes kb-1 .. ke (one plane of redundancy at
//    each chunk end) and B on [kb, ke): planes kb-2 .. ke+1 are staged.  Step m (plane
//    kb-2+m landed) relaxes R1 on plane Q = kb-3+m and, in the same phase by other
//    threads, B on plane Q-2 (whose R1 neighbours were finished one step earlier): one
//    barrier per plane; the rows' codes and f are prefetched before the plane wait.
//  * Rows that are not regular (Gamma_12 / Gamma_F list rows, isoviscous traction-face
//    rows: both couple within a colour) are NOT relaxed here: the caller relaxes the
//    colour-0 list rows from the start-of-pass vector and scatters them into the input
//    before this kernel (so the staged planes already carry their new values), and the
//    colour-1 list rows after it (from this kernel's output: their coefficients to
//    same-colour regular rows are exactly 0).  Dirichlet rows stay 0 (staged as 0).
//  * Output: every owned vertex of the tile (and the face column / row i = n, j = n of
//    the last tiles) is written: B value (colour-1 regular rows) or the staged value.
#pragma once
#include <cstdio>

#include "kernels_tiled.cuh"

namespace stk {

constexpr int SW_TX = 32, SW_TY = 8, SW_NT = SW_TX * SW_TY;
constexpr int SW_BX = SW_TX + 6, SW_BY = SW_TY + 4;   // box: x from i0 - 3 (even start), y ring 2
constexpr int SW_X0 = 3, SW_Y0 = 2;                    // box position of the tile's first column / row
constexpr int SW_PL = SW_BX * SW_BY;                   // 456 doubles
constexpr int SW_FST = ((SW_PL + 15) / 16) * 16;
constexpr int SW_SLOT = 4 * SW_FST;                    // u1, u2, u3, p
constexpr int SW_PREF = 2, SW_RING = 5 + SW_PREF;      // live slots m-4..m + prefetch
constexpr int SW_R1N = (SW_TX + 2) * (SW_TY + 2);      // R1 positions (ring-1 box): 340

struct SweepArgs {
  double* out;          // u_out (3 fields)
  const double* f;      // right-hand side f (fields 0..2)
  int kchunk;
};

// 24 B^T p (unit) by the 7 pair differences D_d = p(v + d) - p(v - d), d in D+ = {x, y, z,
// xy, xz, yz, xyz}: (24 B^T p)_a = sum_d beta^a_d D_d with beta^a_d = 6 (d = e_a), 2 (d_a = 1),
// -2 (d_a = 0), i.e. 8 D_a + 4 (sum of the 3 mixed d with d_a = 1) - 2 sum_d D_d
constexpr bool sw_beta_ok() {
  const int D[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};
  for (int a = 0; a < 3; ++a)
    for (int q = 0; q < 7; ++q) {
      const bool ea = D[q][a] == 1 && D[q][0] + D[q][1] + D[q][2] == 1;
      const int beta = ea ? 6 : D[q][a] == 1 ? 2 : -2;
      if (kst(1, 0, a, 0, D[q][0], D[q][1], D[q][2]) != beta) return false;
      if (kst(1, 0, a, 0, -D[q][0], -D[q][1], -D[q][2]) != -beta) return false;
    }
  return kst(1, 0, 0, 0, 0, 0, 0) == 0 && kst(1, 0, 1, 0, 0, 0, 0) == 0 && kst(1, 0, 2, 0, 0, 0, 0) == 0;
}
static_assert(sw_beta_ok(), "B^T pair factoring disagrees with the Kuhn unit stencils");

// Gauss-Seidel update of the velocity rows of a regular (isoviscous, interior) vertex
// of class `code` at box position s: u += (f - A u - B^T p) / diag(A), A the 7-point
// mu-Laplacian (regular rows of the mod / grad forms) -- the update of
// finish_row<FORM, OP_VEL> (R12) with B^T p pair-factored
template <int FORM>
__device__ __forceinline__ void sw_relax(const DGrid& g, const double* const pl[3], int s, uint8_t code,
                                         const double f[3], double u[3]) {
  static_assert(FORM != FORM_SYM, "the fused sweep needs the 7-point A of the mod / grad forms");
  const double h = g.h;
  const double sA = mu_of(g, code) * h * (1.0 / 6.0), sB = h * h * (1.0 / 24.0);
  const double isA = imu_of(g, code) * (double)g.n * 6.0;
  constexpr double kC = KS<0, FORM_GRAD, 0, 0, 0, 0, 0>::v, kX = KS<0, FORM_GRAD, 0, 0, 1, 0, 0>::v;
  const double* Pm = pl[0] + 3 * SW_FST + s;
  const double* P0 = pl[1] + 3 * SW_FST + s;
  const double* Pp = pl[2] + 3 * SW_FST + s;
  const double Dx = P0[1] - P0[-1], Dy = P0[SW_BX] - P0[-SW_BX], Dz = Pp[0] - Pm[0];
  const double Dxy = P0[SW_BX + 1] - P0[-SW_BX - 1], Dxz = Pp[1] - Pm[-1], Dyz = Pp[SW_BX] - Pm[-SW_BX];
  const double Dxyz = Pp[SW_BX + 1] - Pm[-SW_BX - 1];
  const double S2 = 2.0 * ((Dx + Dy + Dz) + (Dxy + Dxz) + (Dyz + Dxyz));
  const double bt[3] = {fma(8.0, Dx, fma(4.0, Dxy + Dxz + Dxyz, -S2)), fma(8.0, Dy, fma(4.0, Dxy + Dyz + Dxyz, -S2)),
                        fma(8.0, Dz, fma(4.0, Dxz + Dyz + Dxyz, -S2))};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double* q = pl[1] + c * SW_FST + s;
    const double nb = (q[1] + q[-1]) + (q[SW_BX] + q[-SW_BX]) + (pl[0][c * SW_FST + s] + pl[2][c * SW_FST + s]);
    const double A = fma(kC, q[0], kX * nb);
    u[c] = fma(f[c] - fma(sA, A, sB * bt[c]), isA * (1.0 / kC), q[0]);
  }
}

template <int FORM>
__global__ void __launch_bounds__(SW_NT, 2)
    k_fsweep(const __grid_constant__ CUtensorMap mapX, DGrid g, SweepArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem_raw = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + SW_RING * SW_SLOT * sizeof(double));
  constexpr uint32_t TX_BYTES = 4 * SW_PL * sizeof(double);

  const int ntx = g.n / SW_TX, tiles = ntx * (g.n / SW_TY);
  const int tile = blockIdx.x % tiles, chunk = blockIdx.x / tiles;
  const int i0 = (tile % ntx) * SW_TX, j0 = (tile / ntx) * SW_TY;
  const int kb = g.z0 + chunk * a.kchunk;
  const int ke = min(kb + a.kchunk, g.z0 + g.nzl);
  if (kb >= ke) return;
  const int M = ke - kb + 4;  // staged planes kb-2 .. ke+1

  if (threadIdx.x == 0) {
    for (int s = 0; s < SW_RING; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {  // thread 0: stage plane kb-2+q into slot q % RING
    const int s = q % SW_RING;
    const int P = kb - 2 + q;
    fence_proxy_async();
    mbar_expect_tx(&bars[s], TX_BYTES);
    double* dst = ring + s * SW_SLOT;
    // map origin: vertex (-1, -1, z0 - 1); the box starts at vertex (i0 - 3, j0 - 2, P);
    // plane z0 - 2 (read by nobody: R1 is never evaluated on plane z0 - 1 < 1) -> z0 - 1
    const int zc = max(P - g.z0 + 1, 0);
    for (int f = 0; f < 4; ++f) tma_load_4d(dst + f * SW_FST, &mapX, &bars[s], i0 - 2, j0 - 1, zc, f);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < min(SW_RING, M); ++q) issue(q);
  auto slot = [&](int q) { return ring + (q % SW_RING) * SW_SLOT; };

  const int tx = threadIdx.x % SW_TX, ty = threadIdx.x / SW_TX;
  const int it = i0 + tx, jt = j0 + ty;
  const int st = (ty + SW_Y0) * SW_BX + (tx + SW_X0);  // box position of the thread's column
  const bool last_x = i0 + SW_TX == g.n, last_y = j0 + SW_TY == g.n;
  const bool ex_x = last_x && tx == SW_TX - 1, ex_y = last_y && ty == SW_TY - 1;
  const int n = g.n;

  // Dirichlet faces this tile's box touches (block-uniform)
  const unsigned dm = g.dirmask;
  const bool zx0 = (dm & 1u) && i0 == 0, zx1 = (dm & 2u) && last_x;
  const bool zy0 = (dm & 4u) && j0 == 0, zy1 = (dm & 8u) && last_y;
  const bool zxy = zx0 || zx1 || zy0 || zy1;

  // work of the combined phase: red position t < 170 of the ring-1 box (R1) on threads
  // 0..169; black position u < 128 of the tile (B) on threads 170..255 (u < 86) and,
  // second, on threads 0..41 (u = 86..127)
  constexpr int NR = SW_R1N / 2, NB = SW_NT / 2 / 1, NB1 = SW_NT - NR;
  struct Row {
    int i, j, sp;
    bool on;
    uint8_t code;
    double f[3];
  };
  auto r1_row = [&](int Q, Row& w) {  // red position threadIdx.x of plane Q
    const int bj = threadIdx.x / ((SW_TX + 2) / 2);
    w.j = j0 - 1 + bj;
    const int bi = 2 * (threadIdx.x % ((SW_TX + 2) / 2)) + ((i0 - 1 + w.j + Q) & 1);
    w.i = i0 - 1 + bi;
    w.sp = (bj + SW_Y0 - 1) * SW_BX + (bi + SW_X0 - 1);
    w.on = w.i >= 1 && w.j >= 1 && Q >= 1 && w.i < n && w.j < n && Q < n;
  };
  auto b_row = [&](int R, int u, Row& w) {  // black position u of the tile on plane R
    const int bj = u / (SW_TX / 2);
    w.j = j0 + bj;
    const int bi = 2 * (u % (SW_TX / 2)) + ((i0 + w.j + R + 1) & 1);
    w.i = i0 + bi;
    w.sp = (bj + SW_Y0) * SW_BX + (bi + SW_X0);
    w.on = w.i >= 1 && w.j >= 1 && R >= 1 && R < n;
  };
  auto fetch = [&](Row& w, int k) {  // the row's code and f (global, independent of the planes)
    if (!w.on) return;
    const int64_t o = vidx(g, w.i, w.j, k);
    w.code = __ldg(g.code + o);
    w.on = w.code < 0x40;  // list / traction-face rows: relaxed by the caller
    w.f[0] = __ldg(a.f + o);
    w.f[1] = __ldg(a.f + g.fs + o);
    w.f[2] = __ldg(a.f + 2 * g.fs + o);
  };
  auto relax = [&](const Row& w, const double* const pl[3], double* cur) {
    if (!w.on) return;
    double u[3];
    sw_relax<FORM>(g, pl, w.sp, w.code, w.f, u);
#pragma unroll
    for (int c = 0; c < 3; ++c) cur[c * SW_FST + w.sp] = u[c];
  };
  (void)NB;

  // rows of step m (codes and f in registers): fetched one step ahead (software pipeline)
  auto rows_of = [&](int m, Row& w1, Row& w2) {
    const int P = kb - 2 + m, Q = P - 1, R = P - 3;
    const bool doR1 = m >= 2 && m < M, doB = m >= 5 && m <= M;
    w1.on = w2.on = false;
    if (threadIdx.x < NR) {
      if (doR1) {
        r1_row(Q, w1);
        fetch(w1, Q);
      }
      if (doB && threadIdx.x < NB - NB1) {
        b_row(R, NB1 + threadIdx.x, w2);
        fetch(w2, R);
      }
    } else if (doB) {
      b_row(R, threadIdx.x - NR, w2);
      fetch(w2, R);
    }
  };
  Row n1, n2;
  rows_of(0, n1, n2);
  for (int m = 0; m <= M; ++m) {
    const int P = kb - 2 + m, R = P - 3;
    const bool doR1 = m >= 2 && m < M, doB = m >= 5;
    const Row w1 = n1, w2 = n2;
    if (m < M) rows_of(m + 1, n1, n2);
    if (m < M) {
      mbar_wait(&bars[m % SW_RING], (m / SW_RING) & 1);
      double* sl = slot(m);  // velocity of the Dirichlet-face vertices of the landed plane := 0
      const bool zp = ((dm & 16u) && P == 0) || ((dm & 32u) && P == n);
      if (zp) {
        for (int e = threadIdx.x; e < 3 * SW_PL; e += SW_NT) sl[(e / SW_PL) * SW_FST + e % SW_PL] = 0.0;
      } else if (zxy) {
        for (int e = threadIdx.x; e < 3 * (2 * SW_BY + 2 * SW_BX); e += SW_NT) {
          const int c = e / (2 * SW_BY + 2 * SW_BX), r = e % (2 * SW_BY + 2 * SW_BX);
          int bx = -1, by = -1;
          if (r < SW_BY) { if (zx0) { bx = SW_X0; by = r; } }
          else if (r < 2 * SW_BY) { if (zx1) { bx = n - i0 + SW_X0; by = r - SW_BY; } }
          else if (r < 2 * SW_BY + SW_BX) { if (zy0) { by = SW_Y0; bx = r - 2 * SW_BY; } }
          else if (zy1) { by = n - j0 + SW_Y0; bx = r - 2 * SW_BY - SW_BX; }
          if (bx >= 0 && bx < SW_BX && by >= 0 && by < SW_BY) sl[c * SW_FST + by * SW_BX + bx] = 0.0;
        }
      }
      if (zp || zxy) __syncthreads();
    }
    // R1 on plane Q (slots m-2..m, result into m-1) and B on plane R = Q - 2 (slots
    // m-4..m-2, result into m-3): disjoint slots written, every slot read is final
    if (threadIdx.x < NR) {
      if (doR1) {
        const double* pl[3] = {slot(m - 2), slot(m - 1), slot(m)};
        relax(w1, pl, slot(m - 1));
      }
      if (doB) {
        const double* pl[3] = {slot(m - 4), slot(m - 3), slot(m - 2)};
        relax(w2, pl, slot(m - 3));
      }
    } else if (doB) {
      const double* pl[3] = {slot(m - 4), slot(m - 3), slot(m - 2)};
      relax(w2, pl, slot(m - 3));
    }
    __syncthreads();
    if (doB) {  // output of plane R: every column of the tile (+ the face column / row)
      const double* cur = slot(m - 3);
      const int64_t o = vidx(g, it, jt, R);
#pragma unroll
      for (int c = 0; c < 3; ++c) a.out[c * g.fs + o] = cur[c * SW_FST + st];
      if (ex_x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) a.out[c * g.fs + o + 1] = cur[c * SW_FST + st + 1];
      }
      if (ex_y) {
#pragma unroll
        for (int c = 0; c < 3; ++c) a.out[c * g.fs + o + g.px] = cur[c * SW_FST + st + SW_BX];
      }
      if (ex_x && ex_y) {
#pragma unroll
        for (int c = 0; c < 3; ++c) a.out[c * g.fs + o + g.px + 1] = cur[c * SW_FST + st + SW_BX + 1];
      }
    }
    // slot m-4 is free (last read by B of this step); the output above reads slot m-3
    if (threadIdx.x == 0 && m >= 4 && m - 4 + SW_RING < M) issue(m - 4 + SW_RING);
  }
}

inline size_t sweep_smem() { return 1024 + SW_RING * SW_SLOT * sizeof(double) + SW_RING * sizeof(uint64_t); }

inline bool sweep_supported(const DGrid& g) { return g.slipmask == 0 && g.n >= 64 && g.n % SW_TX == 0 && encoder() != nullptr; }

template <int FORM>
bool launch_fsweep_t(const DGrid& g, const double* x, const double* f, double* uout, cudaStream_t st) {
  SweepArgs a{};
  a.out = uout;
  a.f = f;
  // one 4-field map over the stored slab with its ghost frame and halo planes
  CUtensorMap mX;
  if (!make_map(&mX, x, g, 4, -1, g.n, -1, g.n, g.z0 - 1, g.z0 + g.nzl, SW_BX, SW_BY)) return false;
  const size_t sm = sweep_smem();
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_fsweep<FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
      return false;
    attr = true;
  }
  const int tiles = (g.n / SW_TX) * (g.n / SW_TY);
  // chunks long enough that the two redundant R1 planes per chunk stay cheap, enough
  // items for every SM
  int kc = g.nzl >= 256 ? 32 : g.nzl >= 64 ? 16 : 8;
  kc = std::max(1, std::min(kc, g.nzl));
  const int chunks = (g.nzl + kc - 1) / kc;
  a.kchunk = kc;
  k_fsweep<FORM><<<dim3(tiles * chunks), SW_NT, sm, st>>>(mX, g, a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "k_fsweep<%d> n=%d launch: %s\n", FORM, g.n, cudaGetErrorString(e));
  return e == cudaSuccess;
}
// x: the iterate (velocity fields 0..2 and the pressure field 3 of one vector)
inline bool launch_fsweep(int form, const DGrid& g, const double* x, const double* f, double* uout,
                          cudaStream_t st) {
  switch (form) {
    case FORM_MOD: return launch_fsweep_t<FORM_MOD>(g, x, f, uout, st);
    case FORM_GRAD: return launch_fsweep_t<FORM_GRAD>(g, x, f, uout, st);
    default: return false;
  }
}

}  // namespace stk
