// Vector kernels of the outer Krylov iteration (right-preconditioned GMRES(m)
// with the Uzawa V_var cycle as preconditioner).  All loops run
// over the owned vertices of a level vector only (halo planes, ghost frame and
// padding are skipped); reductions are deterministic two-stage sums.
#pragma once
#include "kernels_generic.cuh"

namespace stk {

constexpr int KRY_CHUNK = 16;  // basis vectors per batched dot / update launch

// part[block][q] = sum over owned entries of V_q . w   (q < nv <= KRY_CHUNK, V_q = V + q*vlen);
// with_self: also part[block][KRY_CHUNK] = w . w (the norm of w in the same pass)
__global__ void k_dots(DGrid g, const double* __restrict__ V, int64_t vlen, int nv,
                       const double* __restrict__ w, double* __restrict__ part, int with_self = 0) {
  __shared__ double sh[KRY_CHUNK + 1][32];
  double acc[KRY_CHUNK + 1];
#pragma unroll
  for (int q = 0; q <= KRY_CHUNK; ++q) acc[q] = 0.0;
  int i, j, k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; owned_vertex(g, t, i, j, k);
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = vidx(g, i, j, k);
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double wv = w[f * g.fs + o];
#pragma unroll
      for (int q = 0; q < KRY_CHUNK; ++q)
        if (q < nv) acc[q] += V[q * vlen + f * g.fs + o] * wv;
      if (with_self) acc[KRY_CHUNK] += wv * wv;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q <= KRY_CHUNK; ++q) {
    double v = acc[q];
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    if (lane == 0) sh[q][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x <= KRY_CHUNK) {
    double v = 0.0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += sh[threadIdx.x][w2];
    part[(int64_t)blockIdx.x * (KRY_CHUNK + 1) + threadIdx.x] = v;
  }
}

// out[q] = sum_b part[b][q] in a fixed order (q < nv; with_self: out[nv] = the w.w sum)
__global__ void k_dots_final(const double* __restrict__ part, int nblocks, int nv, double* __restrict__ out,
                             int with_self = 0) {
  const int q = threadIdx.x;
  if (q > nv || (q == nv && !with_self)) return;
  const int src = q < nv ? q : KRY_CHUNK;
  double v = 0.0;
  for (int b = 0; b < nblocks; ++b) v += part[(int64_t)b * (KRY_CHUNK + 1) + src];
  out[q] = v;
}

// w = alpha * w - sum_q c[q] V_q      (owned entries, nv <= KRY_CHUNK)
__global__ void k_update(DGrid g, const double* __restrict__ V, int64_t vlen, int nv,
                         const double* __restrict__ c, double alpha, double* __restrict__ w) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const int64_t o = vidx(g, i, j, k);
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    double v = alpha == 0.0 ? 0.0 : alpha * w[f * g.fs + o];
#pragma unroll
    for (int q = 0; q < KRY_CHUNK; ++q)
      if (q < nv) v -= c[q] * V[q * vlen + f * g.fs + o];
    w[f * g.fs + o] = v;
  }
}

// y = a x + b y  (owned entries)
__global__ void k_axpby(DGrid g, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  int i, j, k;
  if (!owned_vertex(g, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, i, j, k)) return;
  const int64_t o = vidx(g, i, j, k);
#pragma unroll
  for (int f = 0; f < 4; ++f) y[f * g.fs + o] = a * x[f * g.fs + o] + (b == 0.0 ? 0.0 : b * y[f * g.fs + o]);
}

}  // namespace stk

namespace stk {

// ---- fused classical Gram-Schmidt passes over FLAT vectors ---------------------
// Every Krylov vector (residual, basis, A z) is zero outside the owned free entries:
// the kernels that produce them write owned rows only (0 at Dirichlet velocity
// rows) into zero-initialised buffers, and the flat update w - sum c V keeps zeros
// zero.  So the Gram-Schmidt passes run over the whole padded vector as one flat
// double2 stream (no index arithmetic, full coalescing); the zeros add nothing.
constexpr int KRY_MAXV = 32;  // basis vectors per fused pass (GMRES(m) with m + 1 <= 32)
enum { GS_DOTS = 0, GS_UPDATE_DOTS = 1, GS_UPDATE_NORM = 2 };

// MODE GS_DOTS:        part[b][q] = V_q . w               (q < nv), part[b][nv] = w . w
// MODE GS_UPDATE_DOTS: w -= sum_q c[q] V_q;  part[b][q] = V_q . w_new
// MODE GS_UPDATE_NORM: w -= sum_q c[q] V_q;  part[b][0] = w_new . w_new
template <int MODE, int NV>
__global__ void __launch_bounds__(256, 1) k_gs_pass(const double* __restrict__ V, int64_t vlen, int nv,
                                                    double* __restrict__ w, const double* __restrict__ c,
                                                    double* __restrict__ part) {
  constexpr int NA = MODE == GS_UPDATE_NORM ? 1 : NV + 1;
  __shared__ double cs[NV];
  __shared__ double sh[NA][8];
  for (int q = threadIdx.x; q < NV; q += blockDim.x) cs[q] = (MODE != GS_DOTS && q < nv) ? c[q] : 0.0;
  __syncthreads();
  double acc[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) acc[q] = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < vlen; e += (int64_t)gridDim.x * blockDim.x) {
    double x = w[e];
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = q < nv ? __ldcs(V + (int64_t)q * vlen + e) : 0.0;
    if (MODE != GS_DOTS) {
#pragma unroll
      for (int q = 0; q < NV; ++q) x = fma(-cs[q], v[q], x);
      w[e] = x;
    }
    if (MODE == GS_UPDATE_NORM) {
      acc[0] = fma(x, x, acc[0]);
    } else {
#pragma unroll
      for (int q = 0; q < NV; ++q) acc[q] = fma(v[q], x, acc[q]);
      if (MODE == GS_DOTS) acc[NV] = fma(x, x, acc[NV]);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NA; ++q) {
    double s = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sh[q][wid] = s;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NA; q += blockDim.x) {
    double s = 0.0;
    for (int w_ = 0; w_ < (int)(blockDim.x >> 5); ++w_) s += sh[q][w_];
    part[(int64_t)blockIdx.x * (KRY_MAXV + 1) + q] = s;
  }
}

// out[q] = sum_b part[b][q] (fixed order), q < cnt
__global__ void k_gs_final(const double* __restrict__ part, int nblocks, int cnt, double* __restrict__ out) {
  const int q = threadIdx.x;
  if (q >= cnt) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[(int64_t)b * (KRY_MAXV + 1) + q];
  out[q] = s;
}

// y = a x + b y over the flat vector (Krylov vectors only, see above)
__global__ void k_axpby_flat(int64_t vlen, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < vlen; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = a * x[e] + (b == 0.0 ? 0.0 : b * y[e]);
}

}  // namespace stk
