// Z-slab communication: one vertex plane per neighbour per
// exchange, an fp64 allreduce for the norms / gauge sums (once per cycle), the
// agglomeration of the coarsest levels onto every rank, and the one cube layer of
// coarse element data a rank takes from the rank below.  With one rank every call
// is a no-op.
//
// Two backends behind the same calls:
//  * NCCL: one process (rank) per GPU; ncclSend/ncclRecv/ncclBroadcast/ncclAllReduce
//    on the solver stream (the production multi-GPU path over NVLink / NVSwitch).
//  * loopback: P contexts of one process on ONE device, each driven by its own host
//    thread and all on the same CUDA stream (stk_loopback_create).  A collective is a
//    host rendezvous of the P threads: every rank publishes its buffer, then copies
//    from its peers' buffers with one cudaMemcpyAsync per plane or range, then a
//    second rendezvous keeps any rank from enqueueing work that overwrites a buffer
//    before every peer's copy out of it is enqueued (stream order does the rest).  No
//    kernel waits on another.  It makes the P-rank code path (partition, halos, split
//    levels, agglomeration) testable on one GPU: results must equal P = 1 (T4).
#pragma once
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
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
  const unsigned em = elim(gc, I, J, K);
  const int64_t oc = vidx(gc, I, J, K);
  for (int f = 0; f < 4; ++f) {
    if ((em >> f) & 1u) { bc[f * gc.fs + oc] = 0.0; continue; }
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

// loopback allreduce: out = sum over ranks q = 0..P-1 (in that order) of in[q][0..count);
// the rank pointers travel by value in the kernel parameters (no host staging to race on)
constexpr int LB_MAXP = 64;
struct LbPtrs {
  const double* p[LB_MAXP];
};
__global__ void k_loopback_sum(const LbPtrs in, int P, int count, double* __restrict__ out) {
  for (int c = threadIdx.x; c < count; c += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += in.p[q][c];
    out[c] = s;
  }
}

}  // namespace stk

// the loopback group (opaque in stk.h): a host barrier plus published pointers
struct stk_loopback {
  int P = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<void*> ptr;      // published by each rank at a rendezvous
  std::vector<int64_t> aux;    // e.g. the rank's field stride / plane count
  double* dsum = nullptr;      // device result of the allreduce
  void* stream = nullptr;      // the one CUDA stream every rank's context uses
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long gen = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace stk {

#define ST_RET(call)                 \
  do {                               \
    stk_status s__ = (call);         \
    if (s__ != STK_OK) return s__;   \
  } while (0)

struct Comm {
  int rank = 0, nranks = 1;
  stk_loopback* lb = nullptr;
#if STK_HAVE_NCCL
  ncclComm_t nc = nullptr;
#endif

  template <class C>
  stk_status init(C* ctx, int r, int P, const uint8_t* id, stk_loopback* group) {
    rank = r;
    nranks = P;
    if (P == 1) return STK_OK;
    if (group) {
      if (group->P != P) {
        ctx->err = "loopback group size differs from cfg.nranks";
        return STK_EINVAL;
      }
      lb = group;
      return STK_OK;
    }
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

  bool loopback() const { return lb != nullptr; }

  void destroy() {
#if STK_HAVE_NCCL
    if (nc) ncclCommDestroy(nc);
    nc = nullptr;
#endif
  }

  // rendezvous: publish (p, a), wait for all ranks
  void publish(void* p, int64_t a = 0) {
    lb->ptr[rank] = p;
    lb->aux[rank] = a;
    lb->barrier();
  }

  template <class C>
  static stk_status cuda_ok(C* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return STK_OK;
    ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
    return STK_ECUDA;
  }

  // exchange the boundary planes of fields [f0, f0+nf) of a distributed level vector
  // (fs: this rank's field stride; py: plane pitch, equal on all ranks)
  template <class C>
  stk_status halo(C* ctx, int n, int z0, int nzl, int64_t py, int64_t fs, double* v, int f0, int nf,
                  bool replicated) {
    if (nranks == 1 || replicated) return STK_OK;
    (void)n; (void)z0;
    if (lb) {
      // publish (v, fs); a rank's own planes 1..nzl, halos 0 and nzl+1
      publish(v, fs);
      stk_status st = STK_OK;
      for (int f = f0; f < f0 + nf && st == STK_OK; ++f) {
        double* base = v + f * fs;
        if (rank > 0) {  // top owned plane of rank-1 -> my plane 0
          const double* pb = (const double*)lb->ptr[rank - 1] + f * lb->aux[rank - 1];
          // rank-1 owns exactly (n/P) planes (it is not the last rank): its top plane index is that
          st = cuda_ok(ctx, cudaMemcpyAsync(base, pb + (int64_t)nzl_below(n) * py, sizeof(double) * py,
                                            cudaMemcpyDeviceToDevice, ctx->stream), "loopback halo");
        }
        if (st == STK_OK && rank < nranks - 1) {  // first owned plane of rank+1 -> my plane nzl+1
          const double* pa = (const double*)lb->ptr[rank + 1] + f * lb->aux[rank + 1];
          st = cuda_ok(ctx, cudaMemcpyAsync(base + (int64_t)(nzl + 1) * py, pa + py, sizeof(double) * py,
                                            cudaMemcpyDeviceToDevice, ctx->stream), "loopback halo");
        }
      }
      lb->barrier();
      return st;
    }
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
    return STK_OK;
#else
    return STK_EUNSUP;
#endif
  }
  // planes owned by a rank below the last one (the slab partition gives every rank
  // but the last n_l / P planes)
  int nzl_below(int n) const { return n / nranks; }

  // d[0..count) = sum over ranks (count <= 256)
  template <class C>
  stk_status allreduce_sum(C* ctx, double* d, int count) {
    if (nranks == 1) return STK_OK;
    if (lb) {
      publish(d);
      stk_status st = STK_OK;
      if (rank == 0) {
        LbPtrs pt{};
        for (int q = 0; q < nranks; ++q) pt.p[q] = (const double*)lb->ptr[q];
        k_loopback_sum<<<1, 64, 0, ctx->stream>>>(pt, nranks, count, lb->dsum);
        st = cuda_ok(ctx, cudaGetLastError(), "loopback allreduce");
      }
      lb->barrier();  // the sum is enqueued (stream order) before every rank's copy out
      if (st == STK_OK)
        st = cuda_ok(ctx, cudaMemcpyAsync(d, lb->dsum, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream),
                     "loopback allreduce");
      lb->barrier();  // dsum / the pointer table are not reused before every copy is enqueued
      return st;
    }
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

  // every rank holds a buffer of the same layout; rank q owns the byte range
  // [off(q), off(q) + len(q)); afterwards every rank holds every range
  template <class C, class R>
  stk_status allgather_ranges(C* ctx, uint8_t* base, const R& range) {
    if (nranks == 1) return STK_OK;
    if (lb) {
      publish(base);
      stk_status st = STK_OK;
      for (int q = 0; q < nranks && st == STK_OK; ++q) {
        if (q == rank) continue;
        int64_t off, len;
        range(q, off, len);
        if (len <= 0) continue;
        st = cuda_ok(ctx, cudaMemcpyAsync(base + off, (const uint8_t*)lb->ptr[q] + off, (size_t)len,
                                          cudaMemcpyDeviceToDevice, ctx->stream), "loopback gather");
      }
      lb->barrier();
      return st;
    }
#if STK_HAVE_NCCL
    ncclGroupStart();
    for (int q = 0; q < nranks; ++q) {
      int64_t off, len;
      range(q, off, len);
      if (len <= 0) continue;
      ncclBroadcast(base + off, base + off, (size_t)len, ncclUint8, q, nc, ctx->stream);
    }
    ncclResult_t res = ncclGroupEnd();
    if (res != ncclSuccess) {
      ctx->err = std::string("gather: ") + ncclGetErrorString(res);
      return STK_ENCCL;
    }
    return STK_OK;
#else
    return STK_EUNSUP;
#endif
  }

  // rank r < P-1 sends bytes [src_off, src_off + len) of its buffer to rank r+1, which
  // receives them at [0, len) of its own (the lowest stored cube layer)
  template <class C>
  stk_status shift_up(C* ctx, uint8_t* base, int64_t src_off, int64_t len) {
    if (nranks == 1) return STK_OK;
    if (lb) {
      publish(base, src_off);
      stk_status st = STK_OK;
      if (rank > 0)
        st = cuda_ok(ctx, cudaMemcpyAsync(base, (const uint8_t*)lb->ptr[rank - 1] + lb->aux[rank - 1], (size_t)len,
                                          cudaMemcpyDeviceToDevice, ctx->stream), "loopback layer");
      lb->barrier();
      return st;
    }
#if STK_HAVE_NCCL
    ncclGroupStart();
    if (rank < nranks - 1) ncclSend(base + src_off, (size_t)len, ncclUint8, rank + 1, nc, ctx->stream);
    if (rank > 0) ncclRecv(base, (size_t)len, ncclUint8, rank - 1, nc, ctx->stream);
    ncclResult_t res = ncclGroupEnd();
    if (res != ncclSuccess) {
      ctx->err = std::string("layer exchange: ") + ncclGetErrorString(res);
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
    const int P = nranks;
    const int nf = gf.n;
    for (int f = 0; f < 4; ++f) {
      const int64_t fbase = (int64_t)f * gc.fs * 8;
      ST_RET(allgather_ranges(ctx, (uint8_t*)bc, [&](int q, int64_t& off, int64_t& len) {
        int a, b;
        owned_coarse(nf, P, q, a, b);
        off = fbase + (int64_t)(a - gc.z0 + 1) * gc.py * 8;
        len = (int64_t)(b - a) * gc.py * 8;
      }));
    }
    return STK_OK;
  }

  DGrid replicated_view(DGrid gc) const { return gc; }
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
