// The paper's coarse-grid solver, optional
// (stk_set_coarse_solver): on the coarsest level the strain form A_sym replaces
// A_tr, the momentum right-hand side is corrected to r1 + B^T M_L^-1 r2 (reading
// R25: M_L = diag int phi_i / mu, the 1/mu-weighted lumped mass; the sign follows
// from b(v,q) = -(div v, q)), and the system [[A_sym, B^T], [B, -C]] is
// solved by block-diagonal preconditioned MINRES from zero (Elman-Silvester-Wathen
// recurrence): velocity block = `cg_its` steps of Jacobi-preconditioned CG on A_sym,
// pressure block = M_L.  Fixed iteration counts, stop early only when
// gamma_{j+1} <= 1e-14 gamma_1 (reading R24).
//
// One thread-block cluster of CL CTAs runs the whole solve (CL = 1 for n_c = 4, 8
// for n_c = 8, 16 for the paper's n_c = 16): every row of the level carries its
// explicit 4x4-block A_sym stencil (assembled by k_assemble_explicit<FORM_SYM> over
// all vertices), vectors live in a compact field-major scratch [4][V] (vertex t =
// i + (n+1)(j + (n+1)k)) in global memory; phases are separated by cluster barriers
// (release / acquire at cluster scope; vector reads go through L2, ld.global.cg, so no
// SM sees a stale L1 line of another CTA's rows); reductions are fixed-order sums of
// per-CTA partials read through distributed shared memory (deterministic, the same
// bits on every CTA).  A single CTA streams the n_c = 16 stencils (9.6 MB) through one
// SM per operator application; the cluster spreads them over CL SMs.
#pragma once
#include <cooperative_groups.h>
#include "stk_common.cuh"

namespace stk {

constexpr int MR_NT = 512;

struct MinresArgs {
  DGrid g;              // coarsest level (held whole)
  const double* S;      // A_sym explicit stencils [V][EXPL] (rows in vertex order)
  const double* b;      // right-hand side, padded level layout
  double* x;            // solution, padded level layout (all owned entries written)
  double* work;         // scratch: MR_NVEC compact vectors [4][V]
  int its, cg_its;
};
constexpr int MR_NVEC = 14;

__device__ __forceinline__ void mr_coords(const DGrid& g, int t, int& i, int& j, int& k) {
  const int nx = g.n + 1;
  i = t % nx;
  j = (t / nx) % nx;
  k = g.z0 + t / (nx * nx);
}

// work-vector load: through L2 when several CTAs share the vectors
template <int CL>
__device__ __forceinline__ double mr_ld(const double* p) {
  if constexpr (CL > 1) return __ldcg(p);
  else return *p;
}

template <int CL>
__device__ __forceinline__ void mr_bar() {
  if constexpr (CL > 1) cooperative_groups::this_cluster().sync();
  else __syncthreads();
}

// fixed-order sum of v over all threads of the cluster (every thread gets the result);
// slot alternates between calls so one cluster barrier per reduction suffices
template <int CL>
__device__ __forceinline__ double mr_sum(double v, double* red, double* part, int& slot) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  if constexpr (CL == 1) {
    return s;
  } else {
    auto cl = cooperative_groups::this_cluster();
    if (threadIdx.x == 0) part[slot] = s;
    cl.sync();
    double tot = 0.0;
    for (int r = 0; r < CL; ++r) tot += *cl.map_shared_rank(part + slot, r);
    slot ^= 1;
    return tot;
  }
}

// y[r] (rows r in [R0, R1)) = sum over the 15 Kuhn offsets and columns c in [C0, C1)
// of S[t][r][q][c] x[c](t + q), for the rows of vertex t
template <int CL, int R0, int R1, int C0, int C1>
__device__ __forceinline__ void mr_row(const DGrid& g, const double* __restrict__ S, const double* x, int64_t V,
                                       int t, int i, int j, int k, double y[4]) {
  const int nx = g.n + 1;
#pragma unroll
  for (int r = R0; r < R1; ++r) y[r] = 0.0;
  const double* St = S + (int64_t)t * EXPL;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int a = i + kq_dx(q), bq = j + kq_dy(q), c = k + kq_dz(q);
    if (a < 0 || bq < 0 || c < g.z0 || a > g.n || bq > g.n || c >= g.z0 + g.nzl) continue;
    const int tn = a + nx * (bq + nx * (c - g.z0));
#pragma unroll
    for (int cc = C0; cc < C1; ++cc) {
      const double xv = mr_ld<CL>(x + cc * V + tn);
#pragma unroll
      for (int r = R0; r < R1; ++r) y[r] = fma(__ldg(St + (r * NQ + q) * 4 + cc), xv, y[r]);
    }
  }
}

template <int FORM, int CL>
__global__ void __launch_bounds__(MR_NT, 1) k_coarse_minres(const __grid_constant__ MinresArgs A) {
  __shared__ double red[MR_NT / 32];
  __shared__ double part[2];
  int slot = 0;
  const DGrid& g = A.g;
  const int nx = g.n + 1;
  const int64_t V = (int64_t)nx * nx * g.nzl;
  int rank = 0;
  if constexpr (CL > 1) rank = (int)cooperative_groups::this_cluster().block_rank();
  const int tid = rank * blockDim.x + threadIdx.x, nt = CL * blockDim.x;
  double* W = A.work;
  auto vec = [&](int s) { return W + (int64_t)s * 4 * V; };
  auto ld = [&](const double* p) { return mr_ld<CL>(p); };
  // compact vectors: 0 x, 1 v_old, 2 v, 3 v_new, 4 z, 5 z_new, 6 w_old, 7 w, 8 w_new, 9 Kz,
  // 10 ml (field 0) / dinv (fields 1..3), CG: 11 xc, 12 rc, 13 pc (zc in z's fields)
  double* ml = vec(10);
  double* dinv = vec(10) + V;  // [3][V]
  // setup: r = b (compact), ml, dinv; x = v_old = w_old = w = 0
  for (int t = tid; t < V; t += nt) {
    int i, j, k;
    mr_coords(g, t, i, j, k);
    const int64_t o = vidx(g, i, j, k);
    ml[t] = gauge_weight(g, i, j, k);
    const double* inv = A.S + (int64_t)t * EXPL + 4 * NQ * 4;
    for (int f = 0; f < 4; ++f) {
      vec(2)[f * V + t] = A.b[f * g.fs + o];
      vec(0)[f * V + t] = 0.0;
      vec(1)[f * V + t] = 0.0;
      vec(6)[f * V + t] = 0.0;
      vec(7)[f * V + t] = 0.0;
      if (f < 3) dinv[f * V + t] = inv[f];
    }
    // tmp = r_p / ml -> field 3 of vec(9)  (own row)
    vec(9)[3 * V + t] = A.b[3 * g.fs + o] / ml[t];
  }
  mr_bar<CL>();
  // r_u += B^T tmp  (R25)
  for (int t = tid; t < V; t += nt) {
    int i, j, k;
    mr_coords(g, t, i, j, k);
    double y[4];
    mr_row<CL, 0, 3, 3, 4>(g, A.S, vec(9), V, t, i, j, k, y);
    for (int a = 0; a < 3; ++a) vec(2)[a * V + t] += y[a];
  }
  mr_bar<CL>();

  // z = P^-1 v: pressure z_p = v_p / ml; velocity = cg_its Jacobi-PCG steps on A_sym.
  // Reads of another thread's entries only in the operator applications (Pc).
  auto precond = [&](const double* v, double* z) {
    double* xc = vec(11);  // [3][V]
    double* R = vec(12);   // [3][V]
    double* Pc = vec(13);  // [3][V]
    double* Ap = vec(9);   // [3][V] (Kz is not live during precond)
    double* Z = z;         // zc in z's velocity fields until the end
    double rz = 0.0;
    for (int t = tid; t < V; t += nt) {
      for (int a = 0; a < 3; ++a) {
        const double rv = ld(v + a * V + t);
        const double zv = ld(dinv + a * V + t) * rv;
        xc[a * V + t] = 0.0;
        R[a * V + t] = rv;
        Pc[a * V + t] = zv;
        rz = fma(rv, zv, rz);
      }
      z[3 * V + t] = ld(v + 3 * V + t) / ld(ml + t);
    }
    rz = mr_sum<CL>(rz, red, part, slot);  // also the barrier before the Pc reads
    for (int it = 0; it < A.cg_its && rz != 0.0; ++it) {
      double pap = 0.0;
      for (int t = tid; t < V; t += nt) {
        int i, j, k;
        mr_coords(g, t, i, j, k);
        double y[4];
        mr_row<CL, 0, 3, 0, 3>(g, A.S, Pc, V, t, i, j, k, y);
        for (int a = 0; a < 3; ++a) {
          Ap[a * V + t] = y[a];
          pap = fma(ld(Pc + a * V + t), y[a], pap);
        }
      }
      pap = mr_sum<CL>(pap, red, part, slot);
      const double alpha = rz / pap;
      const bool last = it + 1 == A.cg_its;
      double rz_new = 0.0;
      for (int t = tid; t < V; t += nt)
        for (int a = 0; a < 3; ++a) {
          xc[a * V + t] = fma(alpha, ld(Pc + a * V + t), ld(xc + a * V + t));
          const double rv = fma(-alpha, ld(Ap + a * V + t), ld(R + a * V + t));
          R[a * V + t] = rv;
          if (!last) {
            const double zv = ld(dinv + a * V + t) * rv;
            Z[a * V + t] = zv;
            rz_new = fma(rv, zv, rz_new);
          }
        }
      if (last) break;
      rz_new = mr_sum<CL>(rz_new, red, part, slot);  // all Pc reads of this step are done
      const double beta = rz_new / rz;
      for (int t = tid; t < V; t += nt)
        for (int a = 0; a < 3; ++a) Pc[a * V + t] = fma(beta, ld(Pc + a * V + t), ld(Z + a * V + t));
      rz = rz_new;
      mr_bar<CL>();
    }
    for (int t = tid; t < V; t += nt)
      for (int a = 0; a < 3; ++a) z[a * V + t] = ld(xc + a * V + t);
    mr_bar<CL>();
  };

  int ix = 0, iv_old = 1, iv = 2, iv_new = 3, iz = 4, iz_new = 5, iw_old = 6, iw = 7, iw_new = 8;
  precond(vec(iv), vec(iz));
  double zv = 0.0;
  for (int t = tid; t < V; t += nt)
    for (int f = 0; f < 4; ++f) zv = fma(ld(vec(iz) + f * V + t), ld(vec(iv) + f * V + t), zv);
  double gamma = sqrt(fmax(mr_sum<CL>(zv, red, part, slot), 0.0));
  if (gamma > 0.0) {
    const double gamma0 = gamma;
    double gamma_old = 1.0, eta = gamma, s_old = 0.0, s = 0.0, c_old = 1.0, c = 1.0;
    for (int it = 0; it < A.its; ++it) {
      // z /= gamma; Kz = K z; delta = Kz . z
      const double ig = 1.0 / gamma;
      for (int t = tid; t < V; t += nt)
        for (int f = 0; f < 4; ++f) vec(iz)[f * V + t] = ld(vec(iz) + f * V + t) * ig;
      mr_bar<CL>();
      double dl = 0.0;
      for (int t = tid; t < V; t += nt) {
        int i, j, k;
        mr_coords(g, t, i, j, k);
        double y[4];
        mr_row<CL, 0, 4, 0, 4>(g, A.S, vec(iz), V, t, i, j, k, y);
        for (int f = 0; f < 4; ++f) {
          vec(9)[f * V + t] = y[f];
          dl = fma(y[f], ld(vec(iz) + f * V + t), dl);
        }
      }
      const double delta = mr_sum<CL>(dl, red, part, slot);
      const double c1 = delta / gamma, c2 = gamma / gamma_old;
      for (int t = tid; t < V; t += nt)
        for (int f = 0; f < 4; ++f)
          vec(iv_new)[f * V + t] =
              ld(vec(9) + f * V + t) - c1 * ld(vec(iv) + f * V + t) - c2 * ld(vec(iv_old) + f * V + t);
      mr_bar<CL>();
      precond(vec(iv_new), vec(iz_new));
      double zz = 0.0;
      for (int t = tid; t < V; t += nt)
        for (int f = 0; f < 4; ++f) zz = fma(ld(vec(iz_new) + f * V + t), ld(vec(iv_new) + f * V + t), zz);
      const double gamma_new = sqrt(fmax(mr_sum<CL>(zz, red, part, slot), 0.0));
      const double a0 = c * delta - c_old * s * gamma;
      const double a1 = sqrt(a0 * a0 + gamma_new * gamma_new);
      const double a2 = s * delta + c_old * c * gamma;
      const double a3 = s_old * gamma;
      c_old = c;
      s_old = s;
      c = a0 / a1;
      s = gamma_new / a1;
      const double ce = c * eta;
      for (int t = tid; t < V; t += nt)
        for (int f = 0; f < 4; ++f) {
          const double wn =
              (ld(vec(iz) + f * V + t) - a3 * ld(vec(iw_old) + f * V + t) - a2 * ld(vec(iw) + f * V + t)) / a1;
          vec(iw_new)[f * V + t] = wn;
          vec(ix)[f * V + t] = fma(ce, wn, ld(vec(ix) + f * V + t));
        }
      mr_bar<CL>();
      eta = -s * eta;
      int tmp = iv_old;
      iv_old = iv;
      iv = iv_new;
      iv_new = tmp;
      tmp = iw_old;
      iw_old = iw;
      iw = iw_new;
      iw_new = tmp;
      tmp = iz;
      iz = iz_new;
      iz_new = tmp;
      gamma_old = gamma;
      gamma = gamma_new;
      if (gamma <= 1e-14 * gamma0) break;
    }
  }
  // x -> padded level layout (every owned entry; eliminated entries are 0)
  for (int t = tid; t < V; t += nt) {
    int i, j, k;
    mr_coords(g, t, i, j, k);
    const int64_t o = vidx(g, i, j, k);
    for (int f = 0; f < 4; ++f) A.x[f * g.fs + o] = ld(vec(ix) + f * V + t);
  }
  mr_bar<CL>();  // no CTA leaves while another may still read its partials (DSMEM)
}

}  // namespace stk
