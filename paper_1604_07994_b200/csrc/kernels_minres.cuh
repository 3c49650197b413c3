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
// One CTA of MR_NT threads runs the whole solve (the coarsest level has at most a
// few thousand vertices; a multi-CTA version would pay a grid barrier per phase):
// every row of the level carries its explicit 4x4-block A_sym stencil (assembled by
// k_assemble_explicit<FORM_SYM> over all vertices), vectors live in a compact
// field-major scratch [4][V] (vertex t = i + (n+1)(j + (n+1)k)), reductions are
// fixed-order block sums (deterministic).
#pragma once
#include "stk_common.cuh"

namespace stk {

constexpr int MR_NT = 1024;

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

// fixed-order block sum of v over the CTA (all threads get the result)
__device__ __forceinline__ double mr_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// y[r] (rows r in [r0, r1)) = sum over the 15 Kuhn offsets and columns c in [c0, c1)
// of S[t][r][q][c] x[c](t + q), for the rows of vertex t
template <int R0, int R1, int C0, int C1>
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
      const double xv = x[cc * V + tn];
#pragma unroll
      for (int r = R0; r < R1; ++r) y[r] = fma(St[(r * NQ + q) * 4 + cc], xv, y[r]);
    }
  }
}

template <int FORM>
__global__ void __launch_bounds__(MR_NT, 1) k_coarse_minres(const __grid_constant__ MinresArgs A) {
  __shared__ double red[MR_NT / 32];
  const DGrid& g = A.g;
  const int nx = g.n + 1;
  const int64_t V = (int64_t)nx * nx * g.nzl;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* W = A.work;
  auto vec = [&](int s) { return W + (int64_t)s * 4 * V; };
  // compact vectors: 0 x, 1 v_old, 2 v, 3 v_new, 4 z, 5 z_new, 6 w_old, 7 w, 8 w_new, 9 Kz,
  // 10 ml (field 0) / dinv (fields 1..3), CG: 11 xc/rc, 12 zc/pc, 13 Apc
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
  }
  __syncthreads();
  // tmp = r_p / ml -> field 3 of vec(9); then r_u += B^T tmp  (R25)
  for (int t = tid; t < V; t += nt) vec(9)[3 * V + t] = vec(2)[3 * V + t] / ml[t];
  __syncthreads();
  for (int t = tid; t < V; t += nt) {
    int i, j, k;
    mr_coords(g, t, i, j, k);
    double y[4];
    mr_row<0, 3, 3, 4>(g, A.S, vec(9), V, t, i, j, k, y);
    for (int a = 0; a < 3; ++a) vec(2)[a * V + t] += y[a];
  }
  __syncthreads();

  // z = P^-1 v: pressure z_p = v_p / ml; velocity = cg_its Jacobi-PCG steps on A_sym
  auto precond = [&](const double* v, double* z) {
    double* xc = vec(11);            // [3][V] xc
    double* R = vec(12);             // [3][V] rc
    double* Pc = vec(13);            // [3][V] pc
    double* Ap = vec(9);             // [3][V] Apc (Kz is not live during precond)
    double* Z = z;                   // zc kept in z's velocity fields until the end
    double rz = 0.0;
    for (int t = tid; t < V; t += nt) {
      for (int a = 0; a < 3; ++a) {
        const double rv = v[a * V + t];
        const double zv = dinv[a * V + t] * rv;
        xc[a * V + t] = 0.0;
        R[a * V + t] = rv;
        Pc[a * V + t] = zv;
        rz = fma(rv, zv, rz);
      }
      z[3 * V + t] = v[3 * V + t] / ml[t];
    }
    rz = mr_sum(rz, red);
    for (int it = 0; it < A.cg_its && rz != 0.0; ++it) {
      double pap = 0.0;
      for (int t = tid; t < V; t += nt) {
        int i, j, k;
        mr_coords(g, t, i, j, k);
        double y[4];
        mr_row<0, 3, 0, 3>(g, A.S, Pc, V, t, i, j, k, y);
        for (int a = 0; a < 3; ++a) {
          Ap[a * V + t] = y[a];
          pap = fma(Pc[a * V + t], y[a], pap);
        }
      }
      pap = mr_sum(pap, red);
      const double alpha = rz / pap;
      const bool last = it + 1 == A.cg_its;
      double rz_new = 0.0;
      for (int t = tid; t < V; t += nt)
        for (int a = 0; a < 3; ++a) {
          xc[a * V + t] = fma(alpha, Pc[a * V + t], xc[a * V + t]);
          const double rv = fma(-alpha, Ap[a * V + t], R[a * V + t]);
          R[a * V + t] = rv;
          if (!last) {
            const double zv = dinv[a * V + t] * rv;
            Z[a * V + t] = zv;
            rz_new = fma(rv, zv, rz_new);
          }
        }
      if (last) break;
      rz_new = mr_sum(rz_new, red);
      const double beta = rz_new / rz;
      for (int t = tid; t < V; t += nt)
        for (int a = 0; a < 3; ++a) Pc[a * V + t] = fma(beta, Pc[a * V + t], Z[a * V + t]);
      rz = rz_new;
      __syncthreads();
    }
    __syncthreads();
    for (int t = tid; t < V; t += nt)
      for (int a = 0; a < 3; ++a) z[a * V + t] = xc[a * V + t];
    __syncthreads();
  };

  int ix = 0, iv_old = 1, iv = 2, iv_new = 3, iz = 4, iz_new = 5, iw_old = 6, iw = 7, iw_new = 8;
  precond(vec(iv), vec(iz));
  double zv = 0.0;
  for (int t = tid; t < V; t += nt)
    for (int f = 0; f < 4; ++f) zv = fma(vec(iz)[f * V + t], vec(iv)[f * V + t], zv);
  double gamma = sqrt(fmax(mr_sum(zv, red), 0.0));
  if (gamma > 0.0) {
    const double gamma0 = gamma;
    double gamma_old = 1.0, eta = gamma, s_old = 0.0, s = 0.0, c_old = 1.0, c = 1.0;
    for (int it = 0; it < A.its; ++it) {
      // z /= gamma; Kz = K z; delta = Kz . z
      const double ig = 1.0 / gamma;
      for (int t = tid; t < V; t += nt)
        for (int f = 0; f < 4; ++f) vec(iz)[f * V + t] *= ig;
      __syncthreads();
      double dl = 0.0;
      for (int t = tid; t < V; t += nt) {
        int i, j, k;
        mr_coords(g, t, i, j, k);
        double y[4];
        mr_row<0, 4, 0, 4>(g, A.S, vec(iz), V, t, i, j, k, y);
        for (int f = 0; f < 4; ++f) {
          vec(9)[f * V + t] = y[f];
          dl = fma(y[f], vec(iz)[f * V + t], dl);
        }
      }
      const double delta = mr_sum(dl, red);
      const double c1 = delta / gamma, c2 = gamma / gamma_old;
      for (int t = tid; t < V; t += nt)
        for (int f = 0; f < 4; ++f)
          vec(iv_new)[f * V + t] = vec(9)[f * V + t] - c1 * vec(iv)[f * V + t] - c2 * vec(iv_old)[f * V + t];
      __syncthreads();
      precond(vec(iv_new), vec(iz_new));
      double zz = 0.0;
      for (int t = tid; t < V; t += nt)
        for (int f = 0; f < 4; ++f) zz = fma(vec(iz_new)[f * V + t], vec(iv_new)[f * V + t], zz);
      const double gamma_new = sqrt(fmax(mr_sum(zz, red), 0.0));
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
          const double wn = (vec(iz)[f * V + t] - a3 * vec(iw_old)[f * V + t] - a2 * vec(iw)[f * V + t]) / a1;
          vec(iw_new)[f * V + t] = wn;
          vec(ix)[f * V + t] = fma(ce, wn, vec(ix)[f * V + t]);
        }
      __syncthreads();
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
    for (int f = 0; f < 4; ++f) A.x[f * g.fs + o] = vec(ix)[f * V + t];
  }
}

}  // namespace stk
