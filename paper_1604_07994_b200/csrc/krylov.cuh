// Vector kernels of the outer Krylov iteration (right-preconditioned GMRES(m)
// with the Uzawa V_var cycle as preconditioner).  All loops run
// over the owned vertices of a level vector only (halo planes, ghost frame and
// padding are skipped); reductions are deterministic two-stage sums.
#pragma once
#include "kernels_generic.cuh"

namespace stk {

constexpr int KRY_CHUNK = 8;  // basis vectors per batched dot / update launch

// part[block][q] = sum over owned entries of V_q . w   (q < nv <= KRY_CHUNK, V_q = V + q*vlen)
__global__ void k_dots(DGrid g, const double* __restrict__ V, int64_t vlen, int nv,
                       const double* __restrict__ w, double* __restrict__ part) {
  __shared__ double sh[KRY_CHUNK][32];
  double acc[KRY_CHUNK];
#pragma unroll
  for (int q = 0; q < KRY_CHUNK; ++q) acc[q] = 0.0;
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
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < KRY_CHUNK; ++q) {
    double v = acc[q];
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    if (lane == 0) sh[q][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < KRY_CHUNK) {
    double v = 0.0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += sh[threadIdx.x][w2];
    part[(int64_t)blockIdx.x * KRY_CHUNK + threadIdx.x] = v;
  }
}

// out[q] = sum_b part[b][q] in a fixed order
__global__ void k_dots_final(const double* __restrict__ part, int nblocks, int nv, double* __restrict__ out) {
  const int q = threadIdx.x;
  if (q >= nv) return;
  double v = 0.0;
  for (int b = 0; b < nblocks; ++b) v += part[(int64_t)b * KRY_CHUNK + q];
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
