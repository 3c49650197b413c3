// Z-slab communication: one vertex plane per neighbour per
// exchange (ncclSend/ncclRecv in a group on the solver stream), an fp64
// allreduce for the norms / gauge sums (once per cycle), and the agglomeration
// of the coarsest levels onto every rank (each rank broadcasts its planes).
// With one rank every call is a no-op.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/stk.h"
#include "stk_common.cuh"

#if STK_HAVE_NCCL
#include <nccl.h>
#endif

namespace stk {

// restriction into the owned coarse planes of a replicated coarse level:
// like k_restrict but only coarse planes K with 2K owned by this rank
__global__ void k_restrict_part(DGrid gf, DGrid gc, int K0, int K1, const double* __restrict__ rf,
                                double* __restrict__ bc) {
  const int64_t nx = gc.n + 1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nx * nx * (K1 - K0)) return;
  const int I = (int)(t % nx), J = (int)((t / nx) % nx), K = K0 + (int)(t / (nx * nx));
  const int fi = 2 * I, fj = 2 * J, fk = 2 * K;
  const int D[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};
  const bool dir = is_dirichlet(gc, I, J, K);
  const int64_t oc = vidx(gc, I, J, K);
  for (int f = 0; f < 4; ++f) {
    if (f < 3 && dir) { bc[f * gc.fs + oc] = 0.0; continue; }
    const double* r = rf + f * gf.fs;
    double s = r[vidx(gf, fi, fj, fk)];
    double e = 0.0;
    for (int q = 0; q < 7; ++q)
      for (int sg = -1; sg <= 1; sg += 2) {
        const int a = fi + sg * D[q][0], b = fj + sg * D[q][1], c = fk + sg * D[q][2];
        if (a < 0 || b < 0 || c < 0 || a > gf.n || b > gf.n || c > gf.n) continue;
        e += r[vidx(gf, a, b, c)];
      }
    bc[f * gc.fs + oc] = s + 0.5 * e;
  }
}

// coarse classes of the owned coarse cube layers [CK0, CK1) of a replicated level
__global__ void k_coarsen_part(DGrid gf, DGrid gc, int CK0, int CK1, uint8_t* __restrict__ cls_c) {
  const int nc = gc.n;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= (int64_t)(CK1 - CK0) * nc * nc * 6) return;
  const int T = (int)(tid % 6);
  int64_t r = tid / 6;
  const int CI = (int)(r % nc);
  r /= nc;
  const int CJ = (int)(r % nc);
  const int CK = CK0 + (int)(r / nc);
  uint8_t cl[8];
  int cnt[8];
  for (int q = 0; q < 8; ++q) {
    const int off = c_child_off[T][q];
    cl[q] = elem_class(gf, 2 * CI + (off & 1), 2 * CJ + ((off >> 1) & 1), 2 * CK + ((off >> 2) & 1),
                       c_child_t[T][q]);
  }
  for (int q = 0; q < 8; ++q) {
    cnt[q] = 0;
    for (int s = 0; s < 8; ++s) cnt[q] += cl[s] == cl[q];
  }
  int best = 0;
  for (int q = 1; q < 8; ++q) {
    const bool better = cnt[q] > cnt[best] ||
                        (cnt[q] == cnt[best] && (mu_of(gf, cl[q]) > mu_of(gf, cl[best]) ||
                                                 (mu_of(gf, cl[q]) == mu_of(gf, cl[best]) && cl[q] < cl[best])));
    if (better) best = q;
  }
  cls_c[((((int64_t)(CK - gc.cz0)) * nc + CJ) * nc + CI) * 6 + T] = cl[best];
}

struct Comm {
  int rank = 0, nranks = 1;
#if STK_HAVE_NCCL
  ncclComm_t nc = nullptr;
#endif

  template <class C>
  stk_status init(C* ctx, int r, int P, const uint8_t* id) {
    rank = r;
    nranks = P;
    if (P == 1) return STK_OK;
#if STK_HAVE_NCCL
    if (!id) {
      ctx->err = "nranks > 1 needs the NCCL unique id";
      return STK_EINVAL;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclResult_t res = ncclCommInitRank(&nc, P, uid, r);
    if (res != ncclSuccess) {
      ctx->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(res);
      return STK_ENCCL;
    }
    return STK_OK;
#else
    ctx->err = "built without NCCL";
    return STK_EUNSUP;
#endif
  }

  void destroy() {
#if STK_HAVE_NCCL
    if (nc) ncclCommDestroy(nc);
    nc = nullptr;
#endif
  }

  // exchange the boundary planes of fields [f0, f0+nf) of a distributed level vector
  template <class C>
  stk_status halo(C* ctx, int n, int z0, int nzl, int64_t py, int64_t fs, double* v, int f0, int nf,
                  bool replicated) {
    if (nranks == 1 || replicated) return STK_OK;
#if STK_HAVE_NCCL
    ncclGroupStart();
    for (int f = f0; f < f0 + nf; ++f) {
      double* base = v + f * fs;
      if (rank > 0) {
        ncclSend(base + 1 * py, py, ncclDouble, rank - 1, nc, ctx->stream);
        ncclRecv(base + 0 * py, py, ncclDouble, rank - 1, nc, ctx->stream);
      }
      if (rank < nranks - 1) {
        ncclSend(base + (int64_t)nzl * py, py, ncclDouble, rank + 1, nc, ctx->stream);
        ncclRecv(base + (int64_t)(nzl + 1) * py, py, ncclDouble, rank + 1, nc, ctx->stream);
      }
    }
    ncclResult_t res = ncclGroupEnd();
    if (res != ncclSuccess) {
      ctx->err = std::string("halo exchange: ") + ncclGetErrorString(res);
      return STK_ENCCL;
    }
    (void)n; (void)z0;
    return STK_OK;
#else
    return STK_EUNSUP;
#endif
  }

  template <class C>
  stk_status allreduce_sum(C* ctx, double* d, int count) {
    if (nranks == 1) return STK_OK;
#if STK_HAVE_NCCL
    ncclResult_t res = ncclAllReduce(d, d, count, ncclDouble, ncclSum, nc, ctx->stream);
    if (res != ncclSuccess) {
      ctx->err = std::string("allreduce: ") + ncclGetErrorString(res);
      return STK_ENCCL;
    }
    return STK_OK;
#else
    return STK_EUNSUP;
#endif
  }

  // coarse planes [K0,K1) that rank q owns when restricting onto a replicated level
  static void owned_coarse(int nf, int P, int q, int& K0, int& K1) {
    const int per = nf / P;
    const int f0 = q * per, f1 = q * per + per + (q == P - 1 ? 1 : 0);
    K0 = (f0 + 1) / 2;
    K1 = (f1 + 1) / 2;
  }

  template <class C>
  stk_status restrict_to_replicated(C* ctx, DGrid gf, DGrid gc, const double* rf, double* bc) {
    int K0, K1;
    owned_coarse(gf.n, nranks, rank, K0, K1);
    const int64_t nx = gc.n + 1;
    const int64_t work = nx * nx * (K1 - K0);
    if (work > 0) k_restrict_part<<<(unsigned)((work + 255) / 256), 256, 0, ctx->stream>>>(gf, gc, K0, K1, rf, bc);
    ctx->launches++;
#if STK_HAVE_NCCL
    ncclGroupStart();
    for (int q = 0; q < nranks; ++q) {
      int a, b;
      owned_coarse(gf.n, nranks, q, a, b);
      if (b <= a) continue;
      for (int f = 0; f < 4; ++f) {
        double* p = bc + f * gc.fs + (int64_t)(a - gc.z0 + 1) * gc.py;
        ncclBroadcast(p, p, (size_t)(b - a) * gc.py, ncclDouble, q, nc, ctx->stream);
      }
    }
    ncclResult_t res = ncclGroupEnd();
    if (res != ncclSuccess) {
      ctx->err = std::string("coarse gather: ") + ncclGetErrorString(res);
      return STK_ENCCL;
    }
    return STK_OK;
#else
    return nranks == 1 ? STK_OK : STK_EUNSUP;
#endif
  }

  DGrid replicated_view(DGrid gc) const { return gc; }

  template <class C>
  stk_status gather_classes(C* ctx, DGrid gf, DGrid gc, uint8_t* cls_c) {
    // coarse cube layer CK derives from fine cube layers 2CK, 2CK+1: rank q computes
    // the coarse layers whose fine layers it owns, then broadcasts them
    const int nc_ = gc.n;
    const int per = gf.n / nranks;
    const int CK0 = rank * per / 2, CK1 = (rank + 1) * per / 2;
    const int64_t work = (int64_t)(CK1 - CK0) * nc_ * nc_ * 6;
    if (work > 0) k_coarsen_part<<<(unsigned)((work + 255) / 256), 256, 0, ctx->stream>>>(gf, gc, CK0, CK1, cls_c);
    ctx->launches++;
#if STK_HAVE_NCCL
    ncclGroupStart();
    for (int q = 0; q < nranks; ++q) {
      const int a = q * per / 2, b = (q + 1) * per / 2;
      if (b <= a) continue;
      uint8_t* p = cls_c + (int64_t)a * nc_ * nc_ * 6;
      ncclBroadcast(p, p, (size_t)(b - a) * nc_ * nc_ * 6, ncclUint8, q, nc, ctx->stream);
    }
    ncclResult_t res = ncclGroupEnd();
    if (res != ncclSuccess) {
      ctx->err = std::string("class gather: ") + ncclGetErrorString(res);
      return STK_ENCCL;
    }
    return STK_OK;
#else
    return nranks == 1 ? STK_OK : STK_EUNSUP;
#endif
  }
};

inline stk_status comm_unique_id(uint8_t id[128]) {
#if STK_HAVE_NCCL
  ncclUniqueId uid;
  if (ncclGetUniqueId(&uid) != ncclSuccess) return STK_ENCCL;
  memcpy(id, &uid, sizeof(uid) < 128 ? sizeof(uid) : 128);
  return STK_OK;
#else
  (void)id;
  return STK_EUNSUP;
#endif
}

}  // namespace stk
