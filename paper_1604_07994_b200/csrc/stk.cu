// stk.cu — C ABI (include/stk.h) of the B200 Stokes operator / Uzawa multigrid.
//
// One translation unit: the device headers define __constant__ tables that all
// kernels share.  Host code here is setup + launch orchestration only; every
// step of the solver path runs in the kernels of kernels_*.cuh.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/stk.h"
#include "comm.cuh"
#include "kernels_generic.cuh"
#include "kernels_tiled.cuh"
#include "kernels_fused.cuh"
#include "kernels_sweep.cuh"
#include "krylov.cuh"
#include "kernels_minres.cuh"
#include "kernels_p0.cuh"

using namespace stk;

namespace {

struct Level {
  int n = 0;
  double h = 0;
  int z0 = 0, nzl = 0;   // owned vertex planes
  int cz0 = 0, cz1 = 0;  // stored cube layers
  int64_t px = 0, py = 0, fs = 0, vlen = 0;
  uint8_t* cls = nullptr;
  double2* emu = nullptr;  // levels >= 1: per-tet (mu_A, 1/mu_C) means over the Bey children (R15)
  uint8_t* code = nullptr;
  double* x = nullptr;    // MG iterate (levels >= 1)
  double* b = nullptr;    // MG rhs (levels >= 1)
  double* r = nullptr;    // scratch: residual / smoother temporaries
  int64_t nirr = 0;
  int32_t* list = nullptr;  // owned list rows (CODE_IRREGULAR), tiled levels only
  bool replicated = false;  // whole level held by every rank (coarse agglomeration)
  // fused coarse levels (kernels_fused.cuh): explicit stencils of the non-regular rows
  int32_t* slot = nullptr;  // owned linear index -> explicit slot or -1
  int32_t* xrows = nullptr; // explicit rows (owned linear indices)
  double* S = nullptr;      // explicit stencils [slot][EXPL]
  int64_t nexpl = 0;
  double* Slist = nullptr;  // explicit stencils of the list rows [nirr][EXPL] (tiled levels)
  size_t cap_list = 0, cap_Slist = 0, cap_slot = 0, cap_xrows = 0, cap_S = 0;
  // repeat-pass rows (list rows + isoviscous traction-face rows) and their stencils
  int32_t* rlist = nullptr;
  double* Srl = nullptr;
  int64_t nrl = 0;
  size_t cap_rlist = 0, cap_Srl = 0;
  double* cbuf = nullptr;   // in-place velocity passes: results of the repeat-list rows [nrl][3]
  size_t cap_cbuf = 0;
};

// event-timed profile of the kernels launched while enabled (stk_profile_*)
enum { P_APPLY = 0, P_RESID, P_VEL, P_P1, P_P2, P_RESTRICT, P_PROLONG, P_COARSE, P_REDUCE, P_KRYLOV, P_CGRAPH, P_FUSED,
       P_VREP, P_FSWEEP, P_NOPS };
struct ProfRec {
  int op, level;
  cudaEvent_t e0, e1;
};
struct Prof {
  int on = 0;  // 1: per-launch events except inside the coarse graph (timed as one op); 2: no graph
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void reset() {
    for (auto& r : recs) {
      pool.push_back(r.e0);
      pool.push_back(r.e1);
    }
    recs.clear();
  }
  void destroy() {
    reset();
    for (auto e : pool) cudaEventDestroy(e);
    pool.clear();
  }
};

}  // namespace

struct stk_ctx {
  stk_config cfg{};
  cudaStream_t stream = nullptr;
  int nlev = 0;
  std::vector<Level> lev;
  int state = 0;  // 0 created, 1 viscosity set, 2 assembled
  std::vector<double> class_mu;
  std::string err;
  int kernel_mode = 1;
  int64_t launches = 0;
  // coarsest level
  int32_t* cdofs = nullptr;
  int cN = 0, cN1 = 0;
  double* cK = nullptr;
  double* cG = nullptr;
  int* cstatus = nullptr;
  double* d_mu = nullptr;   // per-class mu_k (256) and 1/mu_k (256)
  MuTab mutab{};            // the same table, passed to the row kernels as a parameter
  cudaStream_t side = nullptr;            // list-row kernels run here, forked from `stream`
  cudaStream_t cap = nullptr;             // capture stream for the coarse-level CUDA graph
  cudaGraphExec_t coarse_exec = nullptr;  // levels >= 1 of the V-cycle (fixed internal buffers)
  int64_t coarse_launches = 0;            // kernels in that graph (launch accounting)
  // fused coarse V-cycle (levels fl..nlev-1 in one persistent kernel), fl = -1: off
  int fuse_n = 0;   // 0: fused persistent kernel off (one launch per phase in the graph)
  int fl = -1;
  int row_n = 16;   // levels >= 1 with n_l <= row_n run the row kernels (measured best, cfg2)
  int rl = -1;      // first row level, -1: none
  int fgrid = 0;
  unsigned long long* fbar = nullptr;     // grid-barrier counters (one per prefix size)
  size_t cap_cdofs = 0, cap_cK = 0, cap_cG = 0, cap_cfac = 0;
  unsigned long long* dcnt = nullptr;     // assembly counters (nlev + 1)
  std::vector<int64_t> graph_sig;         // what the captured coarse graph depends on
  FPhase* fprog = nullptr;                // phase program of the fused V-cycle (device)
  int fnph = 0, fgrid_used = 0;
  int fcluster = 0;  // fused V-cycle on one 16-CTA thread-block cluster (cluster barriers)
  double* cfac = nullptr;                 // Gauss-Jordan column factors
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // reductions
  double* part = nullptr;
  double* sums = nullptr;
  double* hsums = nullptr;  // pinned
  int nparts = 0;
  Comm comm;
  Prof prof;
  Prof lvl_pool;          // events around the coarse part of each V-cycle (stk_report.t_level_s)
  int lvl_timing = 0;
  // Krylov workspace (GMRES(m), cfg.krylov = m)
  double* kbasis = nullptr;  // (m+1) level-0 vectors
  double* kwork = nullptr;   // 3 level-0 vectors: w, z, r
  double* kz = nullptr;      // m preconditioned basis vectors Z_j = M^-1 V_j (nullptr: recompute)
  int kz_tried = 0;
  double* kcoef = nullptr;   // device coefficients
  double* kpart = nullptr;   // partial dot products
  // coarsest-level solver: 0 dense inverse of the A_tr system (default), 1 the paper's
  // MINRES on A_sym with the corrected right-hand side (kernels_minres.cuh)
  int coarse_kind = 0, mr_its = 20, mr_cg = 4;
  // P1-P0 solver workspace (stk_p0_solve): composite vectors [level-0 vector | 6 n^3]
  double* p0ws = nullptr;
  size_t cap_p0ws = 0;
  double* mr_S = nullptr;     // A_sym explicit stencils of every coarsest-level vertex
  int32_t* mr_rows = nullptr;
  double* mr_work = nullptr;
  size_t cap_mr_S = 0, cap_mr_rows = 0, cap_mr_work = 0;
};

namespace {
// RAII: brackets the kernel launches of one op with CUDA events when profiling
struct PScope {
  stk_ctx* c;
  int op, lv;
  cudaEvent_t e0 = nullptr;
  PScope(stk_ctx* c_, int op_, int lv_) : c(c_), op(op_), lv(lv_) {
    if (c->prof.on) {
      e0 = c->prof.get();
      cudaEventRecord(e0, c->stream);
    }
  }
  ~PScope() {
    if (c->prof.on && e0) {
      cudaEvent_t e1 = c->prof.get();
      cudaEventRecord(e1, c->stream);
      c->prof.recs.push_back({op, lv, e0, e1});
    }
  }
};
}  // namespace

namespace {

constexpr int kThreads = 256;

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);               \
      return STK_ECUDA;                                                            \
    }                                                                              \
  } while (0)

#define ST(call)                      \
  do {                                \
    stk_status s_ = (call);           \
    if (s_ != STK_OK) return s_;      \
  } while (0)

// device buffer with capacity: reallocated only when it must grow, so re-assembly
// (new viscosity, same grid) keeps every pointer the captured coarse graph holds
template <class T>
bool ensure(T*& p, size_t& cap, size_t count) {
  if (p && count <= cap) return true;
  cudaFree(p);
  p = nullptr;
  cap = 0;
  if (cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)) != cudaSuccess) return false;
  cap = std::max<size_t>(count, 1);
  return true;
}

stk_status launched(stk_ctx* ctx) {
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e);
    return STK_ECUDA;
  }
  return STK_OK;
}

unsigned dirmask_of(const stk_config& c) {
  unsigned m = 0;
  for (int f = 0; f < 6; ++f)
    if (c.face[f] == STK_FACE_DIRICHLET0) m |= 1u << f;
  return m;
}
unsigned slipmask_of(const stk_config& c) {
  unsigned m = 0;
  for (int f = 0; f < 6; ++f)
    if (c.face[f] == STK_FACE_FREESLIP) m |= 1u << f;
  return m;
}

DGrid dgrid(const stk_ctx* ctx, const Level& L) {
  DGrid g;
  g.n = L.n;
  g.z0 = L.z0;
  g.nzl = L.nzl;
  g.cz0 = L.cz0;
  g.px = L.px;
  g.py = L.py;
  g.fs = L.fs;
  g.h = L.h;
  g.delta = ctx->cfg.delta;
  g.idh3 = 1.0 / (ctx->cfg.delta * L.h * L.h * L.h);
  g.dirmask = dirmask_of(ctx->cfg);
  g.slipmask = slipmask_of(ctx->cfg);
  g.cls = L.cls;
  g.emu = L.emu;
  g.code = L.code;
  g.mu = ctx->d_mu;
  return g;
}

int64_t owned_vertices(const Level& L) { return (int64_t)(L.n + 1) * (L.n + 1) * L.nzl; }
unsigned nblocks(int64_t work) { return (unsigned)((work + kThreads - 1) / kThreads); }
// small levels (n <= 16): one warp per row (latency-bound; kernels_generic.cuh *_gw)
bool warp_rows(const Level& L) {
  static const int gw_n = getenv("STK_GW_N") ? atoi(getenv("STK_GW_N")) : 16;
  return L.n <= gw_n;
}
unsigned nblocks_gw(const Level& L) { return (unsigned)((owned_vertices(L) * 32 + GW_NT - 1) / GW_NT); }

bool has_traction(const stk_config& c) {
  for (int f = 0; f < 6; ++f)
    if (c.face[f] == STK_FACE_TRACTION) return true;
  return false;
}

void host_tables(int8_t perm[6][3], int8_t corner[8][6], int8_t choff[6][8], int8_t cht[6][8]) {
  const int P[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  for (int t = 0; t < 6; ++t) {
    for (int d = 0; d < 3; ++d) perm[t][d] = (int8_t)P[t][d];
    // vertex offsets a0..a3 as corner bits
    int a[4];
    a[0] = 0;
    a[1] = 1 << P[t][0];
    a[2] = a[1] | (1 << P[t][1]);
    a[3] = 7;
    for (int c = 0; c < 8; ++c) {
      corner[c][t] = -1;
      for (int m = 0; m < 4; ++m)
        if (a[m] == c) corner[c][t] = (int8_t)m;
    }
  }
  // Bey children: fine tet (cube offset o, type t) lies in coarse tet T iff its
  // centroid q (coarse-cube units) satisfies q[sT1] > q[sT2] > q[sT3].
  for (int T = 0; T < 6; ++T) {
    int cnt = 0;
    for (int o = 0; o < 8; ++o)
      for (int t = 0; t < 6; ++t) {
        double q[3];
        for (int d = 0; d < 3; ++d) q[d] = (o >> d) & 1;
        q[P[t][0]] += 0.75;
        q[P[t][1]] += 0.5;
        q[P[t][2]] += 0.25;
        for (int d = 0; d < 3; ++d) q[d] *= 0.5;
        if (q[P[T][0]] > q[P[T][1]] && q[P[T][1]] > q[P[T][2]]) {
          choff[T][cnt] = (int8_t)o;
          cht[T][cnt] = (int8_t)t;
          ++cnt;
        }
      }
    if (cnt != 8) fprintf(stderr, "stk: Bey child table broken (%d)\n", cnt);
  }
}

// ---- z-slab partition of the level hierarchy (host only) ------
// Rank r of P owns vertex planes [r n_l/P, (r+1) n_l/P) of level l (the last rank
// also k = n_l) and the cube layers its stars touch.  A level is distributed
// while n_l/P >= 2 and it is not the coarsest; once a level is replicated every
// coarser one is too (whole level on every rank, restriction gathers it).
struct SlabLevel {
  int n, z0, nzl, cz0, cz1, replicated, K0, K1;  // K0/K1: owned planes of the next (replicated) level, or -1
};
void slab_partition(int n, int nc, int P, int rank, std::vector<SlabLevel>& out) {
  out.clear();
  for (int m = n; m >= nc; m /= 2) out.push_back(SlabLevel{m, 0, 0, 0, 0, 0, -1, -1});
  const int nlev = (int)out.size();
  for (int l = 0; l < nlev; ++l) {
    SlabLevel& L = out[l];
    L.replicated = !(P == 1 || (L.n % P == 0 && L.n / P >= 2 && l < nlev - 1));
    if (l > 0 && out[l - 1].replicated) L.replicated = 1;
    const int r = L.replicated ? 0 : rank;
    const int Pn = L.replicated ? 1 : P;
    const int per = L.n / Pn;
    L.z0 = r * per;
    L.nzl = per + (r == Pn - 1 ? 1 : 0);
    L.cz0 = std::max(0, L.z0 - 1);
    L.cz1 = std::min(L.n, L.z0 + L.nzl);
  }
  for (int l = 0; l + 1 < nlev; ++l)
    if (!out[l].replicated && out[l + 1].replicated) Comm::owned_coarse(out[l].n, P, rank, out[l].K0, out[l].K1);
}

// ---- level operations ------------------------------------------------------

ListView lview(const stk_ctx* ctx, const Level& L) {
  static const bool xl = !getenv("STK_LIST_EXPLICIT") || atoi(getenv("STK_LIST_EXPLICIT"));
  return ListView{L.list, (int)L.nirr, xl ? L.Slist : nullptr, ctx->side, ctx->ev_fork, ctx->ev_join};
}

bool use_tiled(const stk_ctx* ctx, const Level& L) {
  return ctx->kernel_mode == 1 && L.n >= 64 && !L.replicated && tiled_supported(L.n);
}

stk_status op_apply(stk_ctx* ctx, int l, unsigned blocks, const double* x, double* y) {
  Level& L = ctx->lev[l];
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, const_cast<double*>(x), 0, 4, L.replicated));
  DGrid g = dgrid(ctx, L);
  PScope ps(ctx, P_APPLY, l);
  if (use_tiled(ctx, L)) {
    ST(launch_apply_tiled(ctx->cfg.form, g, lview(ctx, L), x, y, blocks, ctx->stream) ? STK_OK : STK_EUNSUP);
    return launched(ctx);
  }
  if (warp_rows(L)) {
    const unsigned nw = nblocks_gw(L);
    switch (ctx->cfg.form) {
      case FORM_MOD: k_apply_gw<FORM_MOD><<<nw, GW_NT, 0, ctx->stream>>>(g, x, y, blocks); break;
      case FORM_SYM: k_apply_gw<FORM_SYM><<<nw, GW_NT, 0, ctx->stream>>>(g, x, y, blocks); break;
      default: k_apply_gw<FORM_GRAD><<<nw, GW_NT, 0, ctx->stream>>>(g, x, y, blocks); break;
    }
    return launched(ctx);
  }
  const unsigned nb = nblocks(owned_vertices(L));
  switch (ctx->cfg.form) {
    case FORM_MOD: k_apply_generic<FORM_MOD><<<nb, kThreads, 0, ctx->stream>>>(g, x, y, blocks); break;
    case FORM_SYM: k_apply_generic<FORM_SYM><<<nb, kThreads, 0, ctx->stream>>>(g, x, y, blocks); break;
    default: k_apply_generic<FORM_GRAD><<<nb, kThreads, 0, ctx->stream>>>(g, x, y, blocks); break;
  }
  return launched(ctx);
}

stk_status op_residual(stk_ctx* ctx, int l, const double* x, const double* b, double* r) {
  Level& L = ctx->lev[l];
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, const_cast<double*>(x), 0, 4, L.replicated));
  DGrid g = dgrid(ctx, L);
  PScope ps(ctx, P_RESID, l);
  if (use_tiled(ctx, L)) {
    ST(launch_residual_tiled(ctx->cfg.form, g, lview(ctx, L), x, b, r, ctx->stream) ? STK_OK : STK_EUNSUP);
    return launched(ctx);
  }
  if (warp_rows(L)) {
    const unsigned nw = nblocks_gw(L);
    switch (ctx->cfg.form) {
      case FORM_MOD: k_residual_gw<FORM_MOD><<<nw, GW_NT, 0, ctx->stream>>>(g, x, b, r); break;
      case FORM_SYM: k_residual_gw<FORM_SYM><<<nw, GW_NT, 0, ctx->stream>>>(g, x, b, r); break;
      default: k_residual_gw<FORM_GRAD><<<nw, GW_NT, 0, ctx->stream>>>(g, x, b, r); break;
    }
    return launched(ctx);
  }
  const unsigned nb = nblocks(owned_vertices(L));
  switch (ctx->cfg.form) {
    case FORM_MOD: k_residual_generic<FORM_MOD><<<nb, kThreads, 0, ctx->stream>>>(g, x, b, r); break;
    case FORM_SYM: k_residual_generic<FORM_SYM><<<nb, kThreads, 0, ctx->stream>>>(g, x, b, r); break;
    default: k_residual_generic<FORM_GRAD><<<nb, kThreads, 0, ctx->stream>>>(g, x, b, r); break;
  }
  return launched(ctx);
}

// one Uzawa step in place on x (4 fields), rhs b; scratch L.r
stk_status op_uzawa(stk_ctx* ctx, int l, double* x, const double* b) {
  Level& L = ctx->lev[l];
  DGrid g = dgrid(ctx, L);
  const int nc = ctx->cfg.ncolors_u;
  const unsigned nb = nblocks(owned_vertices(L));
  double* tmp = L.r;  // fields 0..2: velocity ping-pong, field 3: pressure temp T
  double* p = x + 3 * L.fs;
  const bool tiled = use_tiled(ctx, L);
  // pressure halo is fixed during the velocity sweep
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, x, 3, 1, L.replicated));
  static const bool inplace_env = !getenv("STK_VEL_INPLACE") || atoi(getenv("STK_VEL_INPLACE"));
  // the fused forward sweep (kernels_sweep.cuh) is exact and parity-tested, but measured
  // slower than the in-place colour passes on B200 (cfg3 n = 256: 648 us vs 2 x 320 us plus
  // un-overlapped list passes): opt-in with STK_FSWEEP=1
  static const bool fsweep_env = getenv("STK_FSWEEP") && atoi(getenv("STK_FSWEEP"));
  if (tiled && fsweep_env && ctx->cfg.form != FORM_SYM && nc == 2 && ctx->cfg.nranks == 1 && L.Srl &&
      sweep_supported(g)) {
    // symmetric sweep 0, 1, (1), 0 (R12) with the forward half fused into one pass
    // (kernels_sweep.cuh): colour-0 list rows -> k_fsweep (x -> tmp) -> colour-1 list rows
    // -> repeat of the colour-1 list rows -> colour-0 pass (tmp -> x)
    ListView rv = lview(ctx, L);
    rv.list = L.rlist;
    rv.n = (int)L.nrl;
    rv.S = L.Srl;
    {
      PScope ps(ctx, P_VREP, l);
      ST(launch_vel_inplace(ctx->cfg.form, g, rv, x, p, b, L.cbuf, 0, nc, true, ctx->stream) ? STK_OK : STK_EUNSUP);
      ST(launched(ctx));
    }
    {
      PScope ps(ctx, P_FSWEEP, l);
      ST(launch_fsweep(ctx->cfg.form, g, x, b, tmp, ctx->stream) ? STK_OK : STK_EUNSUP);
      ST(launched(ctx));
    }
    {
      PScope ps(ctx, P_VREP, l);
      ST(launch_vel_inplace(ctx->cfg.form, g, rv, tmp, p, b, L.cbuf, 1, nc, true, ctx->stream) ? STK_OK : STK_EUNSUP);
      ST(launch_vel_inplace(ctx->cfg.form, g, rv, tmp, p, b, L.cbuf, 1, nc, true, ctx->stream) ? STK_OK : STK_EUNSUP);
      ST(launched(ctx));
    }
    {
      PScope ps(ctx, P_VEL, l);
      ST(launch_vel_pass_tiled(ctx->cfg.form, g, lview(ctx, L), tmp, p, b, x, 0, nc, ctx->stream) ? STK_OK
                                                                                               : STK_EUNSUP);
      ST(launched(ctx));
    }
  } else if (tiled && inplace_env && ctx->cfg.form != FORM_SYM && L.Srl) {
    // in-place colour passes 0, 1, (1: list rows only), 0 -- see launch_vel_inplace
    ListView rv = lview(ctx, L);
    rv.list = L.rlist;
    rv.n = (int)L.nrl;
    rv.S = L.Srl;
    for (int s = 0; s < 2 * nc; ++s) {
      const int color = s < nc ? s : 2 * nc - 1 - s;
      const bool list_only = s == nc;
      ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, x, 0, 3, L.replicated));
      PScope ps(ctx, list_only ? P_VREP : P_VEL, l);
      ST(launch_vel_inplace(ctx->cfg.form, g, rv, x, p, b, L.cbuf, color, nc, list_only, ctx->stream) ? STK_OK
                                                                                                   : STK_EUNSUP);
      ST(launched(ctx));
    }
  } else {
  int pass = 0;
  for (int s = 0; s < 2 * nc; ++s, ++pass) {
    const int color = s < nc ? s : 2 * nc - 1 - s;
    const double* uin = (pass & 1) ? tmp : x;
    double* uout = (pass & 1) ? x : tmp;
    ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, const_cast<double*>(uin), 0, 3, L.replicated));
    static const bool repeat_env = !getenv("STK_VEL_REPEAT") || atoi(getenv("STK_VEL_REPEAT"));
    // second pass of the middle colour pair: list + traction-face rows only (forms whose
    // regular rows have a diagonal centre block: mod, grad; the sym centre block
    // couples the 3 components of a vertex, so its repeat is not a no-op)
    const bool repeat = tiled && s == nc && repeat_env && ctx->cfg.form != FORM_SYM;
    PScope ps(ctx, repeat ? P_VREP : P_VEL, l);
    if (repeat) {
      ListView rv = lview(ctx, L);
      rv.list = L.rlist;
      rv.n = (int)L.nrl;
      rv.S = L.Srl;
      ST(launch_vel_repeat(ctx->cfg.form, g, rv, uin, p, b, uout, color, nc, ctx->stream) ? STK_OK : STK_EUNSUP);
    } else if (tiled) {
      ST(launch_vel_pass_tiled(ctx->cfg.form, g, lview(ctx, L), uin, p, b, uout, color, nc, ctx->stream) ? STK_OK
                                                                                           : STK_EUNSUP);
    } else if (warp_rows(L)) {
      const unsigned nw = nblocks_gw(L);
      switch (ctx->cfg.form) {
        case FORM_MOD: k_vel_pass_gw<FORM_MOD><<<nw, GW_NT, 0, ctx->stream>>>(g, uin, p, b, uout, color, nc); break;
        case FORM_SYM: k_vel_pass_gw<FORM_SYM><<<nw, GW_NT, 0, ctx->stream>>>(g, uin, p, b, uout, color, nc); break;
        default: k_vel_pass_gw<FORM_GRAD><<<nw, GW_NT, 0, ctx->stream>>>(g, uin, p, b, uout, color, nc); break;
      }
    } else {
      switch (ctx->cfg.form) {
        case FORM_MOD: k_vel_pass_generic<FORM_MOD><<<nb, kThreads, 0, ctx->stream>>>(g, uin, p, b, uout, color, nc); break;
        case FORM_SYM: k_vel_pass_generic<FORM_SYM><<<nb, kThreads, 0, ctx->stream>>>(g, uin, p, b, uout, color, nc); break;
        default: k_vel_pass_generic<FORM_GRAD><<<nb, kThreads, 0, ctx->stream>>>(g, uin, p, b, uout, color, nc); break;
      }
    }
    ST(launched(ctx));
  }
  }
  // 2*nc passes: result is back in x
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, x, 0, 3, L.replicated));
  double* T = tmp + 3 * L.fs;
  const double* gp = b + 3 * L.fs;
  {
  PScope ps(ctx, P_P1, l);
  if (tiled) {
    ST(launch_p_pass1_tiled(ctx->cfg.form, g, lview(ctx, L), x, gp, T, ctx->stream) ? STK_OK : STK_EUNSUP);
  } else if (warp_rows(L)) {
    const unsigned nw = nblocks_gw(L);
    switch (ctx->cfg.form) {
      case FORM_MOD: k_p_pass1_gw<FORM_MOD><<<nw, GW_NT, 0, ctx->stream>>>(g, x, gp, T); break;
      case FORM_SYM: k_p_pass1_gw<FORM_SYM><<<nw, GW_NT, 0, ctx->stream>>>(g, x, gp, T); break;
      default: k_p_pass1_gw<FORM_GRAD><<<nw, GW_NT, 0, ctx->stream>>>(g, x, gp, T); break;
    }
  } else {
    switch (ctx->cfg.form) {
      case FORM_MOD: k_p_pass1_generic<FORM_MOD><<<nb, kThreads, 0, ctx->stream>>>(g, x, gp, T); break;
      case FORM_SYM: k_p_pass1_generic<FORM_SYM><<<nb, kThreads, 0, ctx->stream>>>(g, x, gp, T); break;
      default: k_p_pass1_generic<FORM_GRAD><<<nb, kThreads, 0, ctx->stream>>>(g, x, gp, T); break;
    }
  }
  ST(launched(ctx));
  }
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, tmp, 3, 1, L.replicated));
  PScope ps2(ctx, P_P2, l);
  if (tiled) {
    ST(launch_p_pass2_tiled(ctx->cfg.form, g, lview(ctx, L), T, p, ctx->cfg.omega, ctx->stream) ? STK_OK : STK_EUNSUP);
  } else if (warp_rows(L)) {
    k_p_pass2_gw<FORM_MOD><<<nblocks_gw(L), GW_NT, 0, ctx->stream>>>(g, T, p, ctx->cfg.omega);
  } else {
    k_p_pass2_generic<FORM_MOD><<<nb, kThreads, 0, ctx->stream>>>(g, T, p, ctx->cfg.omega);
  }
  return launched(ctx);
}

stk_status op_restrict(stk_ctx* ctx, int lf, const double* rf, double* bc) {
  Level& F = ctx->lev[lf];
  Level& C = ctx->lev[lf + 1];
  ST(ctx->comm.halo(ctx, F.n, F.z0, F.nzl, F.py, F.fs, const_cast<double*>(rf), 0, 4, F.replicated));
  if (C.replicated && !F.replicated) {
    // distributed fine level -> replicated coarse level: restrict locally into the
    // owned coarse planes, then gather the coarse planes of all ranks
    ST(ctx->comm.restrict_to_replicated(ctx, dgrid(ctx, F), dgrid(ctx, C), rf, bc));
    return STK_OK;
  }
  PScope ps(ctx, P_RESTRICT, lf);
  k_restrict<<<nblocks(owned_vertices(C)), kThreads, 0, ctx->stream>>>(dgrid(ctx, F), dgrid(ctx, C), rf, bc);
  return launched(ctx);
}

stk_status op_prolong_add(stk_ctx* ctx, int lc, const double* xc, double* xf) {
  Level& C = ctx->lev[lc];
  Level& F = ctx->lev[lc - 1];
  ST(ctx->comm.halo(ctx, C.n, C.z0, C.nzl, C.py, C.fs, const_cast<double*>(xc), 0, 4, C.replicated));
  DGrid gc = dgrid(ctx, C);
  if (C.replicated && !F.replicated) gc = ctx->comm.replicated_view(gc);
  PScope ps(ctx, P_PROLONG, lc);
  k_prolong_add<<<nblocks(owned_vertices(F)), kThreads, 0, ctx->stream>>>(gc, dgrid(ctx, F), xc, xf);
  return launched(ctx);
}

stk_status op_coarse_minres(stk_ctx* ctx, const double* b, double* x) {
  Level& L = ctx->lev[ctx->nlev - 1];
  MinresArgs A{};
  A.g = dgrid(ctx, L);
  A.S = ctx->mr_S;
  A.b = b;
  A.x = x;
  A.work = ctx->mr_work;
  A.its = ctx->mr_its;
  A.cg_its = ctx->mr_cg;
  PScope ps(ctx, P_COARSE, ctx->nlev - 1);
  const int64_t V = owned_vertices(L);
  // one cluster: 1 CTA (n_c = 4), 8 (n_c = 8), 16 (n_c = 16, non-portable size)
  const int cl = V <= 256 ? 1 : V <= 1500 ? 8 : 16;
  if (cl == 1) {
    k_coarse_minres<FORM_SYM, 1><<<1, MR_NT, 0, ctx->stream>>>(A);
    return launched(ctx);
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(cl);
  lc.blockDim = dim3(MR_NT);
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (cl == 8) {
    CK(cudaLaunchKernelEx(&lc, k_coarse_minres<FORM_SYM, 8>, A));
  } else {
    CK(cudaFuncSetAttribute(k_coarse_minres<FORM_SYM, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaLaunchKernelEx(&lc, k_coarse_minres<FORM_SYM, 16>, A));
  }
  return launched(ctx);
}

stk_status op_coarse(stk_ctx* ctx, const double* b, double* x) {
  if (ctx->coarse_kind == 1) return op_coarse_minres(ctx, b, x);
  Level& L = ctx->lev[ctx->nlev - 1];
  const size_t sh = sizeof(double) * ctx->cN;
  if (sh > 48 * 1024) {  // n_coarse = 8 / 16: opt in to the large dynamic shared memory
    if (sh > 227 * 1024) {
      ctx->err = "coarse right-hand side exceeds shared memory (n_coarse too large for op_coarse)";
      return STK_EUNSUP;
    }
    CK(cudaFuncSetAttribute(k_coarse_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  }
  PScope ps(ctx, P_COARSE, ctx->nlev - 1);
  k_coarse_apply<<<1, 1024, sh, ctx->stream>>>(dgrid(ctx, L), ctx->cdofs, ctx->cN, ctx->cN1, ctx->cG, b, x);
  return launched(ctx);
}

// squared norms (+ gauge sums) of a level vector, summed over ranks, into ctx->sums (device)
stk_status op_partials(stk_ctx* ctx, int l, const double* x, int with_gauge) {
  Level& L = ctx->lev[l];
  DGrid g = dgrid(ctx, L);
  PScope ps(ctx, P_REDUCE, l);
  k_partials<<<ctx->nparts, 256, 0, ctx->stream>>>(g, x, ctx->part, with_gauge);
  ST(launched(ctx));
  k_partials_final<<<1, 256, 0, ctx->stream>>>(ctx->part, ctx->nparts, ctx->sums);
  ST(launched(ctx));
  if (!L.replicated) ST(ctx->comm.allreduce_sum(ctx, ctx->sums, 6));
  return STK_OK;
}

stk_status op_gauge(stk_ctx* ctx, int l, double* x) {
  if (has_traction(ctx->cfg)) return STK_OK;
  Level& L = ctx->lev[l];
  ST(op_partials(ctx, l, x, 1));
  k_gauge_apply<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), x, ctx->sums);
  return launched(ctx);
}

stk_status op_vcycle(stk_ctx* ctx, int l, const double* b, double* x);

// ---- row kernels of the context-owned coarse levels (kernels_fused.cuh) ---------
bool row_level(const stk_ctx* ctx, int l) { return l >= 1 && l >= ctx->rl && ctx->rl > 0; }
FLevel flevel(const stk_ctx* ctx, int l) {
  const Level& L = ctx->lev[l];
  FLevel F{};
  F.g = dgrid(ctx, L);
  F.x = L.x;
  F.b = L.b;
  F.r = L.r;
  F.slot = L.slot;
  F.S = L.S;
  return F;
}
template <int OP, int LPR>
void launch_rowl(stk_ctx* ctx, const FLevel& F, const FLevel& F2, int64_t rows, const double* uin, double* uout,
                 int color) {
  const unsigned nb = (unsigned)((rows * LPR + ROW_NT - 1) / ROW_NT);
  const int nc = ctx->cfg.ncolors_u;
  const double om = ctx->cfg.omega;
  switch (ctx->cfg.form) {
    case FORM_MOD: k_rowl<FORM_MOD, OP, LPR><<<nb, ROW_NT, 0, ctx->stream>>>(F, F2, uin, uout, color, nc, om, ctx->mutab); break;
    case FORM_SYM: k_rowl<FORM_SYM, OP, LPR><<<nb, ROW_NT, 0, ctx->stream>>>(F, F2, uin, uout, color, nc, om, ctx->mutab); break;
    default: k_rowl<FORM_GRAD, OP, LPR><<<nb, ROW_NT, 0, ctx->stream>>>(F, F2, uin, uout, color, nc, om, ctx->mutab); break;
  }
}
// lanes per row: 16 (one Kuhn offset per lane) on the latency-bound small levels,
// 4 on larger ones (fewer shuffles per row); STK_ROW_LPR overrides
template <int OP>
stk_status launch_row(stk_ctx* ctx, const FLevel& F, const FLevel& F2, int64_t rows, const double* uin = nullptr,
                      double* uout = nullptr, int color = 0) {
  static const int env = getenv("STK_ROW_LPR") ? atoi(getenv("STK_ROW_LPR")) : 0;
  // chosen from the level's GLOBAL size (not the rows this rank owns): the lane split
  // fixes the summation order, so every partition gives the same bits
  const int64_t gv = (int64_t)(F.g.n + 1) * (F.g.n + 1) * (F.g.n + 1);
  const int lpr = env == 1 || env == 4 || env == 8 || env == 16 ? env : (gv <= 40000 ? 16 : 4);
  (void)rows;
  if (lpr == 16) launch_rowl<OP, 16>(ctx, F, F2, rows, uin, uout, color);
  else if (lpr == 8) launch_rowl<OP, 8>(ctx, F, F2, rows, uin, uout, color);
  else if (lpr == 4) launch_rowl<OP, 4>(ctx, F, F2, rows, uin, uout, color);
  else {
    const unsigned nb = (unsigned)((rows + ROW_NT - 1) / ROW_NT);
    const int nc = ctx->cfg.ncolors_u;
    const double om = ctx->cfg.omega;
    switch (ctx->cfg.form) {
      case FORM_MOD: k_row<FORM_MOD, OP><<<nb, ROW_NT, 0, ctx->stream>>>(F, F2, uin, uout, color, nc, om); break;
      case FORM_SYM: k_row<FORM_SYM, OP><<<nb, ROW_NT, 0, ctx->stream>>>(F, F2, uin, uout, color, nc, om); break;
      default: k_row<FORM_GRAD, OP><<<nb, ROW_NT, 0, ctx->stream>>>(F, F2, uin, uout, color, nc, om); break;
    }
  }
  return launched(ctx);
}
// one Uzawa step on a row level, in place on L.x with rhs L.b (as op_uzawa)
stk_status op_uzawa_rows(stk_ctx* ctx, int l) {
  Level& L = ctx->lev[l];
  const FLevel F = flevel(ctx, l);
  const int64_t V = owned_vertices(L);
  const int nc = ctx->cfg.ncolors_u;
  double* x = L.x;
  double* tmp = L.r;
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, x, 3, 1, L.replicated));
  for (int s = 0; s < 2 * nc; ++s) {
    const int color = s < nc ? s : 2 * nc - 1 - s;
    const double* uin = (s & 1) ? tmp : x;
    double* uout = (s & 1) ? x : tmp;
    ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, const_cast<double*>(uin), 0, 3, L.replicated));
    PScope ps(ctx, P_VEL, l);
    ST(launch_row<FPH_VEL>(ctx, F, F, V, uin, uout, color));
  }
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, x, 0, 3, L.replicated));
  {
    PScope ps(ctx, P_P1, l);
    ST(launch_row<FPH_P1>(ctx, F, F, V));
  }
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, tmp, 3, 1, L.replicated));
  PScope ps(ctx, P_P2, l);
  return launch_row<FPH_P2>(ctx, F, F, V);
}
stk_status op_residual_rows(stk_ctx* ctx, int l) {
  Level& L = ctx->lev[l];
  ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, L.x, 0, 4, L.replicated));
  PScope ps(ctx, P_RESID, l);
  return launch_row<FPH_RES>(ctx, flevel(ctx, l), flevel(ctx, l), owned_vertices(L));
}
// b_c = R r_f and x_c = 0 (both levels row levels, no agglomeration step between)
stk_status op_restrict_rows(stk_ctx* ctx, int lf) {
  Level& F = ctx->lev[lf];
  ST(ctx->comm.halo(ctx, F.n, F.z0, F.nzl, F.py, F.fs, F.r, 0, 4, F.replicated));
  PScope ps(ctx, P_RESTRICT, lf);
  return launch_row<FPH_RESTRICT>(ctx, flevel(ctx, lf), flevel(ctx, lf + 1), owned_vertices(ctx->lev[lf + 1]));
}
stk_status op_prolong_rows(stk_ctx* ctx, int lc) {
  Level& C = ctx->lev[lc];
  ST(ctx->comm.halo(ctx, C.n, C.z0, C.nzl, C.py, C.fs, C.x, 0, 4, C.replicated));
  PScope ps(ctx, P_PROLONG, lc);
  return launch_row<FPH_PROLONG>(ctx, flevel(ctx, lc - 1), flevel(ctx, lc), owned_vertices(ctx->lev[lc - 1]));
}
stk_status op_coarse_rows(stk_ctx* ctx) {
  if (ctx->coarse_kind == 1) {
    Level& L = ctx->lev[ctx->nlev - 1];
    return op_coarse_minres(ctx, L.b, L.x);
  }
  PScope ps(ctx, P_COARSE, ctx->nlev - 1);
  k_coarse_warp<<<(ctx->cN + 7) / 8, 256, 0, ctx->stream>>>(flevel(ctx, ctx->nlev - 1), ctx->cdofs, ctx->cG, ctx->cN,
                                                           ctx->cN1);
  return launched(ctx);
}

// V-cycle of the fused levels fl..nlev-1 on lev[fl].b (x from 0) in one persistent
// cooperative kernel (kernels_fused.cuh)
template <int FORM>
stk_status launch_fused_t(stk_ctx* ctx) {
  FusedArgs A{};
  A.nl = ctx->nlev - ctx->fl;
  for (int q = 0; q < A.nl; ++q) {
    Level& L = ctx->lev[ctx->fl + q];
    FLevel& F = A.L[q];
    F.g = dgrid(ctx, L);
    F.x = L.x;
    F.b = L.b;
    F.r = L.r;
    F.slot = L.slot;
    F.S = L.S;
  }
  A.nph = ctx->fnph;
  A.prog = ctx->fprog;
  A.ncolors = ctx->cfg.ncolors_u;
  A.omega = ctx->cfg.omega;
  A.cdofs = ctx->cdofs;
  A.cG = ctx->cG;
  A.cN = ctx->cN;
  A.cld = ctx->cN1;
  A.bar = ctx->fbar;
  cudaLaunchConfig_t lc{};
  A.cluster = ctx->fcluster;
  lc.gridDim = dim3(ctx->fcluster ? FCL : ctx->fgrid_used);
  lc.blockDim = dim3(256);
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  if (ctx->fcluster) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = FCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    CK(cudaFuncSetAttribute(k_mg_fused<FORM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  } else {
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  }
  lc.attrs = at;
  lc.numAttrs = 1;
  static const bool trace = getenv("STK_FUSED_TRACE") && atoi(getenv("STK_FUSED_TRACE"));
  static unsigned long long* tbuf = nullptr;
  if (trace && !tbuf) CK(cudaMallocManaged(&tbuf, sizeof(unsigned long long) * (FPH_MAX + 1)));
  A.trace = trace ? tbuf : nullptr;
  CK(cudaLaunchKernelEx(&lc, k_mg_fused<FORM>, A));
  if (trace) {  // debug: per-phase durations (CTA 0 clock after each phase's barrier)
    CK(cudaStreamSynchronize(ctx->stream));
    static const char* nm[] = {"zero", "vel", "p1", "p2", "resid", "restrict", "prolong", "coarse"};
    std::vector<FPhase> hp(ctx->fnph);
    CK(cudaMemcpy(hp.data(), ctx->fprog, sizeof(FPhase) * ctx->fnph, cudaMemcpyDeviceToHost));
    std::vector<std::pair<std::string, std::pair<double, int>>> agg;
    unsigned long long prev = tbuf[FPH_MAX];
    for (int k = 0; k < ctx->fnph; ++k) {
      const double dt = (tbuf[k] - prev) * 1e-3;
      prev = tbuf[k];
      const std::string key = "L" + std::to_string(hp[k].lev) + " " + nm[hp[k].op] + " m=" + std::to_string(hp[k].m);
      bool found = false;
      for (auto& e : agg)
        if (e.first == key) { e.second.first += dt; e.second.second++; found = true; }
      if (!found) agg.push_back({key, {dt, 1}});
    }
    for (auto& e : agg)
      fprintf(stderr, "  %-24s %4d x %8.2f us = %9.1f us\n", e.first.c_str(), e.second.second,
              e.second.first / e.second.second, e.second.first);
  }
  return launched(ctx);
}
stk_status op_fused(stk_ctx* ctx) {
  PScope ps(ctx, P_FUSED, ctx->fl);
  switch (ctx->cfg.form) {
    case FORM_MOD: return launch_fused_t<FORM_MOD>(ctx);
    case FORM_SYM: return launch_fused_t<FORM_SYM>(ctx);
    default: return launch_fused_t<FORM_GRAD>(ctx);
  }
}

// lev[1].x = V-cycle of levels >= 1 on lev[1].b from a zero guess.  These
// levels only touch context-owned buffers, so the whole sequence (a few hundred
// small launches with the V_var schedule) is captured once into a CUDA graph
// and replayed; the graph is rebuilt after every stk_assemble.
stk_status op_coarse_part_impl(stk_ctx* ctx);
// levels >= 1 of the V-cycle, bracketed by events while stk_solve collects t_level_s
stk_status op_coarse_part(stk_ctx* ctx) {
  if (!ctx->lvl_timing) return op_coarse_part_impl(ctx);
  cudaEvent_t e0 = ctx->lvl_pool.get(), e1 = ctx->lvl_pool.get();
  CK(cudaEventRecord(e0, ctx->stream));
  const stk_status s = op_coarse_part_impl(ctx);
  CK(cudaEventRecord(e1, ctx->stream));
  ctx->lvl_pool.recs.push_back({P_CGRAPH, 1, e0, e1});
  return s;
}
stk_status op_coarse_part_impl(stk_ctx* ctx) {
  Level& C = ctx->lev[1];
  static const bool no_graph = getenv("STK_NO_GRAPH") && atoi(getenv("STK_NO_GRAPH"));
  if (ctx->fl == 1) return op_fused(ctx);  // one launch: nothing to capture
  // (the loopback exchanger's host rendezvous cannot be captured: launch directly)
  if (ctx->prof.on == 2 || no_graph || ctx->comm.loopback()) {
    CK(cudaMemsetAsync(C.x, 0, sizeof(double) * C.vlen, ctx->stream));
    return op_vcycle(ctx, 1, C.b, C.x);
  }
  if (!ctx->coarse_exec) {
    const int prof_saved = ctx->prof.on;
    ctx->prof.on = 0;  // no timing events inside the captured graph
    cudaStream_t saved = ctx->stream;
    ctx->stream = ctx->cap;
    CK(cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeRelaxed));
    const int64_t l0 = ctx->launches;
    stk_status s = STK_OK;
    if (cudaMemsetAsync(C.x, 0, sizeof(double) * C.vlen, ctx->cap) != cudaSuccess) s = STK_ECUDA;
    if (s == STK_OK) s = op_vcycle(ctx, 1, C.b, C.x);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->cap, &graph);
    ctx->stream = saved;
    ctx->prof.on = prof_saved;
    ctx->coarse_launches = ctx->launches - l0;  // counted when the graph is launched
    ctx->launches = l0;
    if (s != STK_OK) return s;
    if (e != cudaSuccess) {
      ctx->err = std::string("coarse graph capture: ") + cudaGetErrorString(e);
      return STK_ECUDA;
    }
    const cudaError_t ei = cudaGraphInstantiate(&ctx->coarse_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
      ctx->coarse_exec = nullptr;
      ctx->err = std::string("coarse graph instantiate: ") + cudaGetErrorString(ei);
      return STK_ECUDA;
    }
  }
  {
    PScope ps(ctx, P_CGRAPH, 1);
    CK(cudaGraphLaunch(ctx->coarse_exec, ctx->stream));
  }
  ctx->launches += ctx->coarse_launches;
  return STK_OK;
}

// V_var cycle (R13) on level l.  Levels >= 1 are context-owned
// (b = lev[l].b, x = lev[l].x); row levels (n_l <= row_n) run the lean row kernels.
stk_status op_vcycle(stk_ctx* ctx, int l, const double* b, double* x) {
  if (l == ctx->nlev - 1) return row_level(ctx, l) ? op_coarse_rows(ctx) : op_coarse(ctx, b, x);
  Level& L = ctx->lev[l];
  Level& C = ctx->lev[l + 1];
  const bool rows = row_level(ctx, l);
  const int nu_pre = ctx->cfg.nu_pre + ctx->cfg.nu_inc * l;
  const int nu_post = ctx->cfg.nu_post + ctx->cfg.nu_inc * l;
  for (int s = 0; s < nu_pre; ++s) ST(rows ? op_uzawa_rows(ctx, l) : op_uzawa(ctx, l, x, b));
  ST(rows ? op_residual_rows(ctx, l) : op_residual(ctx, l, x, b, L.r));
  const bool rows_tr = rows && row_level(ctx, l + 1) && (C.replicated == L.replicated);
  ST(rows_tr ? op_restrict_rows(ctx, l) : op_restrict(ctx, l, L.r, C.b));
  if (l == 0) {
    ST(op_coarse_part(ctx));
  } else if (l + 1 == ctx->fl) {
    ST(op_fused(ctx));
  } else {
    if (!rows_tr) CK(cudaMemsetAsync(C.x, 0, sizeof(double) * C.vlen, ctx->stream));
    ST(op_vcycle(ctx, l + 1, C.b, C.x));
  }
  ST(rows_tr ? op_prolong_rows(ctx, l + 1) : op_prolong_add(ctx, l + 1, C.x, x));
  for (int s = 0; s < nu_post; ++s) ST(rows ? op_uzawa_rows(ctx, l) : op_uzawa(ctx, l, x, b));
  return STK_OK;
}

// ---- outer Krylov iteration ----------------------------------------------------

constexpr int kDotBlocks = 296;

// dev out[q] = <V_q, w> over owned entries, all ranks (stream-ordered, no host sync);
// with_self: also out[nv] = <w, w> (fused into the first chunk's pass)
stk_status op_dots_dev(stk_ctx* ctx, const double* V, int nv, const double* w, double* out, int with_self = 0) {
  Level& L = ctx->lev[0];
  DGrid g = dgrid(ctx, L);
  PScope ps(ctx, P_KRYLOV, 0);
  for (int c0 = 0; c0 < nv; c0 += KRY_CHUNK) {
    const int m = std::min(KRY_CHUNK, nv - c0);
    const int ws = (with_self && c0 == 0) ? 1 : 0;
    k_dots<<<kDotBlocks, 256, 0, ctx->stream>>>(g, V + (int64_t)c0 * L.vlen, L.vlen, m, w, ctx->kpart, ws);
    ST(launched(ctx));
    k_dots_final<<<1, 32, 0, ctx->stream>>>(ctx->kpart, kDotBlocks, m, out + c0, 0);
    ST(launched(ctx));
    if (ws) {  // the w.w sum of the same pass -> out[nv]
      k_dots_final<<<1, 32, 0, ctx->stream>>>(ctx->kpart, kDotBlocks, 0, out + nv, 1);
      ST(launched(ctx));
    }
  }
  if (!L.replicated) ST(ctx->comm.allreduce_sum(ctx, out, nv + (with_self ? 1 : 0)));
  return STK_OK;
}

// one fused Gram-Schmidt pass over the flat basis V(0..nv-1) (krylov.cuh); `cnt`
// results into out (device), summed over ranks
constexpr int kGsBlocks = 296;
template <int MODE>
stk_status op_gs(stk_ctx* ctx, const double* V, int nv, double* w, const double* c, double* out, int cnt) {
  Level& L = ctx->lev[0];
  PScope ps(ctx, P_KRYLOV, 0);
  if (nv <= 8) k_gs_pass<MODE, 8><<<kGsBlocks, 256, 0, ctx->stream>>>(V, L.vlen, nv, w, c, ctx->kpart);
  else if (nv <= 16) k_gs_pass<MODE, 16><<<kGsBlocks, 256, 0, ctx->stream>>>(V, L.vlen, nv, w, c, ctx->kpart);
  else k_gs_pass<MODE, 32><<<kGsBlocks, 256, 0, ctx->stream>>>(V, L.vlen, nv, w, c, ctx->kpart);
  ST(launched(ctx));
  k_gs_final<<<1, 64, 0, ctx->stream>>>(ctx->kpart, kGsBlocks, cnt, out);
  ST(launched(ctx));
  if (!L.replicated) ST(ctx->comm.allreduce_sum(ctx, out, cnt));
  return STK_OK;
}

// host out[q] = <V_q, w> (synchronises)
stk_status op_dots(stk_ctx* ctx, const double* V, int nv, const double* w, double* out) {
  ST(op_dots_dev(ctx, V, nv, w, ctx->kcoef));
  CK(cudaMemcpyAsync(out, ctx->kcoef, sizeof(double) * nv, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return STK_OK;
}

// w = alpha w - sum_q c[q] V_q, coefficients c on the device
stk_status op_update_dev(stk_ctx* ctx, const double* V, int nv, const double* c, double alpha, double* w) {
  Level& L = ctx->lev[0];
  DGrid g = dgrid(ctx, L);
  PScope ps(ctx, P_KRYLOV, 0);
  for (int c0 = 0; c0 < nv || c0 == 0; c0 += KRY_CHUNK) {
    const int m = std::min(KRY_CHUNK, nv - c0);
    k_update<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(g, V + (int64_t)c0 * L.vlen, L.vlen, m,
                                                                         c + c0, c0 == 0 ? alpha : 1.0, w);
    ST(launched(ctx));
    if (nv == 0) break;
  }
  return STK_OK;
}

// w = alpha w - sum_q c[q] V_q  (c on the host)
stk_status op_update(stk_ctx* ctx, const double* V, int nv, const double* c, double alpha, double* w) {
  CK(cudaMemcpyAsync(ctx->kcoef, c, sizeof(double) * nv, cudaMemcpyHostToDevice, ctx->stream));
  return op_update_dev(ctx, V, nv, ctx->kcoef, alpha, w);
}

stk_status op_vcycle(stk_ctx* ctx, int l, const double* b, double* x);

// Right-preconditioned restarted GMRES(m) on K x = b with M^-1 = one V_var cycle
// from a zero guess (a fixed linear map).  CGS2 orthogonalisation, Givens rotations;
// the preconditioned vectors Z_j = M^-1 V_j are kept (m more level-0 vectors) so the
// restart correction is x += Z y; without the memory, x += M^-1 (V y) costs one extra
// cycle per restart.
stk_status op_gmres(stk_ctx* ctx, const double* b, double* x, double rtol, int max_its, stk_report* R,
                    double bnorm, int& its, double& rel) {
  Level& L = ctx->lev[0];
  const int m = ctx->cfg.krylov;
  const int64_t vlen = L.vlen;
  const size_t vb = sizeof(double) * vlen;
  if (!ctx->kbasis) {
    if (cudaMalloc(&ctx->kbasis, vb * (m + 1)) != cudaSuccess || cudaMalloc(&ctx->kwork, vb * 3) != cudaSuccess ||
        cudaMalloc(&ctx->kcoef, sizeof(double) * (4 * (m + 2) + KRY_CHUNK)) != cudaSuccess ||
        cudaMalloc(&ctx->kpart, sizeof(double) * std::max(kDotBlocks * (KRY_CHUNK + 1),
                                                           kGsBlocks * (KRY_MAXV + 1))) != cudaSuccess) {
      cudaGetLastError();
      ctx->err = "out of device memory for the GMRES basis (reduce cfg.krylov)";
      return STK_ENOMEM;
    }
    CK(cudaMemsetAsync(ctx->kbasis, 0, vb * (m + 1), ctx->stream));
    CK(cudaMemsetAsync(ctx->kwork, 0, vb * 3, ctx->stream));
  }
  // keep Z_j = M^-1 V_j when the memory is there: the restart update is then x += Z y
  // (no extra preconditioner cycle per restart); else x += M^-1 (V y)
  if (!ctx->kz && !ctx->kz_tried) {
    ctx->kz_tried = 1;
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    if (vb * (size_t)m + (size_t)(2u << 30) < fr && cudaMalloc(&ctx->kz, vb * m) != cudaSuccess) {
      cudaGetLastError();
      ctx->kz = nullptr;
    }
  }
  double* w = ctx->kwork;
  double* z = ctx->kwork + vlen;
  double* r = ctx->kwork + 2 * vlen;
  auto V = [&](int q) { return ctx->kbasis + (int64_t)q * vlen; };
  auto Zv = [&](int q) { return ctx->kz ? ctx->kz + (int64_t)q * vlen : z; };
  DGrid g0 = dgrid(ctx, L);
  const unsigned nb = nblocks(owned_vertices(L));
  std::vector<double> H((m + 1) * m, 0.0), cs(m), sn(m), gv(m + 1), h(m + 1), h2(m + 1), y(m);
  double nr;
  ST(op_residual(ctx, 0, x, b, r));
  ST(op_dots(ctx, r, 1, r, &nr));
  double beta = std::sqrt(nr);
  rel = bnorm > 0 ? beta / bnorm : 0.0;
  while (rel > rtol && its < max_its) {
    k_axpby_flat<<<kGsBlocks, 256, 0, ctx->stream>>>(vlen, 1.0 / beta, r, 0.0, V(0));
    ST(launched(ctx));
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int jdone = 0;
    for (int j = 0; j < m && its < max_its; ++j) {
      double* zj = Zv(j);
      CK(cudaMemsetAsync(zj, 0, vb, ctx->stream));
      ST(op_vcycle(ctx, 0, V(j), zj));
      ST(op_apply(ctx, 0, BLK_ALL, zj, w));
      if (m + 1 <= KRY_MAXV) {
        // classical Gram-Schmidt twice (CGS2) in three fused flat passes: dots; update +
        // the second pass's dots; update + ||w||^2 -- one host round trip per iteration.
        // (CGS1 with the Pythagorean norm, two passes, measured 34 instead of 29 GMRES
        // iterations on cfg3 n = 256: the lost orthogonality costs more than the pass.)
        double* c1 = ctx->kcoef + (m + 2);
        double* c2 = ctx->kcoef + 2 * (m + 2);
        double* nw = ctx->kcoef + 3 * (m + 2);
        ST(op_gs<GS_DOTS>(ctx, V(0), j + 1, w, nullptr, c1, j + 1));
        ST(op_gs<GS_UPDATE_DOTS>(ctx, V(0), j + 1, w, c1, c2, j + 1));
        ST(op_gs<GS_UPDATE_NORM>(ctx, V(0), j + 1, w, c2, nw, 1));
        std::vector<double> hc(3 * (m + 2));
        CK(cudaMemcpyAsync(hc.data(), c1, sizeof(double) * 3 * (m + 2), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (int q = 0; q <= j; ++q) h[q] = hc[q] + hc[(m + 2) + q];
        h[j + 1] = std::sqrt(std::max(hc[2 * (m + 2)], 0.0));
      } else {
        // long restarts: chunked CGS2 with the coefficients on the device
        double* c1 = ctx->kcoef + (m + 2);
        double* c2 = ctx->kcoef + 2 * (m + 2);
        ST(op_dots_dev(ctx, V(0), j + 1, w, c1, 0));
        ST(op_update_dev(ctx, V(0), j + 1, c1, 1.0, w));
        ST(op_dots_dev(ctx, V(0), j + 1, w, c2, 0));
        ST(op_update_dev(ctx, V(0), j + 1, c2, 1.0, w));
        ST(op_dots_dev(ctx, w, 1, w, c2 + (j + 1), 0));
        std::vector<double> hc(2 * (m + 2));
        CK(cudaMemcpyAsync(hc.data(), c1, sizeof(double) * 2 * (m + 2), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (int q = 0; q <= j; ++q) h[q] = hc[q] + hc[(m + 2) + q];
        h[j + 1] = std::sqrt(std::max(hc[(m + 2) + j + 1], 0.0));
      }
      if (h[j + 1] > 0) {
        k_axpby_flat<<<kGsBlocks, 256, 0, ctx->stream>>>(vlen, 1.0 / h[j + 1], w, 0.0, V(j + 1));
        ST(launched(ctx));
      }
      for (int q = 0; q < j; ++q) {  // previous rotations
        const double t = cs[q] * h[q] + sn[q] * h[q + 1];
        h[q + 1] = -sn[q] * h[q] + cs[q] * h[q + 1];
        h[q] = t;
      }
      const double den = std::hypot(h[j], h[j + 1]);
      cs[j] = den > 0 ? h[j] / den : 1.0;
      sn[j] = den > 0 ? h[j + 1] / den : 0.0;
      h[j] = den;
      h[j + 1] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      for (int q = 0; q <= j; ++q) H[q * m + j] = h[q];
      ++its;
      jdone = j + 1;
      rel = bnorm > 0 ? std::fabs(gv[j + 1]) / bnorm : 0.0;
      if (its < 256) R->res_hist[its] = rel;
      if (!std::isfinite(rel)) {
        R->nan_seen = 1;
        return STK_OK;
      }
      if (rel <= rtol) break;
    }
    // y = H^-1 g (upper triangular), x += M^-1 (V y)
    for (int q = jdone - 1; q >= 0; --q) {
      double s = gv[q];
      for (int c = q + 1; c < jdone; ++c) s -= H[q * m + c] * y[c];
      y[q] = s / H[q * m + q];
    }
    for (int q = 0; q < jdone; ++q) y[q] = -y[q];
    if (ctx->kz) {
      ST(op_update(ctx, ctx->kz, jdone, y.data(), 1.0, x));  // x += sum y_q Z_q
    } else {
      ST(op_update(ctx, V(0), jdone, y.data(), 0.0, w));  // w = sum y_q V_q
      CK(cudaMemsetAsync(z, 0, vb, ctx->stream));
      ST(op_vcycle(ctx, 0, w, z));
      k_axpby<<<nb, kThreads, 0, ctx->stream>>>(g0, 1.0, z, 1.0, x);
      ST(launched(ctx));
    }
    ST(op_residual(ctx, 0, x, b, r));
    ST(op_dots(ctx, r, 1, r, &nr));
    beta = std::sqrt(nr);
    rel = bnorm > 0 ? beta / bnorm : 0.0;  // true residual after the restart
    if (its < 256) R->res_hist[its] = rel;
  }
  return STK_OK;
}

// persistent-grid size (one 256-thread CTA per SM) and the barrier words
stk_status fused_setup(stk_ctx* ctx) {
  // the fused V-cycle (off by default, stk_set_fuse_n) on one 16-CTA cluster with hardware
  // cluster barriers (STK_FUSED_CLUSTER=1) or on a cooperative grid with the software grid
  // barrier over the participating CTA prefix (default: faster for the one-CTA phases of
  // the n <= 8 levels; cfg3 n = 256, fuse_n = 8: 16.3 vs 16.7 ms per cycle; both slower than
  // the graph of per-phase launches, 15.96 ms, profiles/r02_levels_fused_cluster.log)
  static const bool cl_env = getenv("STK_FUSED_CLUSTER") && atoi(getenv("STK_FUSED_CLUSTER"));
  ctx->fcluster = cl_env ? 1 : 0;
  if (!ctx->fbar) {
    int dev = 0, nsm = 0, per = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mg_fused<FORM_SYM>, 256, 0));
    int per2 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_gauss_jordan_coop, 256, 0));
    per = std::min(per, per2);
    ctx->fgrid = std::max(1, nsm * std::max(1, per));
    const size_t words = (size_t)(ctx->fgrid + 2);
    CK(cudaMalloc(&ctx->fbar, sizeof(unsigned long long) * words));
    CK(cudaMemsetAsync(ctx->fbar, 0, sizeof(unsigned long long) * words, ctx->stream));
  }
  return STK_OK;
}

// first fused level: n_l <= fuse_n, below the finest, every level from there
// on held whole by this rank; explicit stencils of its non-regular rows
stk_status fused_assemble(stk_ctx* ctx) {
  ctx->fl = -1;
  for (auto& L : ctx->lev) L.nexpl = 0;
  ctx->rl = -1;
  if (ctx->kernel_mode != 1) return STK_OK;
  int rl = -1;
  for (int l = 1; l < ctx->nlev; ++l)
    if (ctx->lev[l].n <= ctx->row_n) {
      rl = l;
      break;
    }
  if (rl < 0) return STK_OK;
  int fl = -1;
  if (ctx->fuse_n > 0 && ctx->coarse_kind == 0)
    for (int l = ctx->nlev - 2; l >= rl; --l) {
      const Level& L = ctx->lev[l];
      if (L.n > ctx->fuse_n || (ctx->cfg.nranks > 1 && !L.replicated) || ctx->nlev - l > FMAX) break;
      fl = l;
    }
  ST(assemble_stencils(ctx->stream) ? STK_OK : STK_ECUDA);
  if (!ctx->dcnt) CK(cudaMalloc(&ctx->dcnt, sizeof(unsigned long long) * (ctx->nlev + 1)));
  unsigned long long* dcnt = ctx->dcnt + ctx->nlev;
  for (int l = rl; l < ctx->nlev; ++l) {
    Level& L = ctx->lev[l];
    const int64_t V = owned_vertices(L);
    if (!ensure(L.slot, L.cap_slot, (size_t)L.fs) || !ensure(L.xrows, L.cap_xrows, (size_t)V)) return STK_ENOMEM;
    CK(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long), ctx->stream));
    k_build_explicit<<<nblocks(V), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), L.slot, L.xrows, dcnt);
    ST(launched(ctx));
    unsigned long long c = 0;
    CK(cudaMemcpyAsync(&c, dcnt, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    L.nexpl = (int64_t)c;
    if (c == 0) continue;
    if (!ensure(L.S, L.cap_S, (size_t)EXPL * c)) return STK_ENOMEM;
    const unsigned nb = nblocks((int64_t)c * NQ * 4);
    DGrid g = dgrid(ctx, L);
    switch (ctx->cfg.form) {
      case FORM_MOD: k_assemble_explicit<FORM_MOD><<<nb, kThreads, 0, ctx->stream>>>(g, L.xrows, (int)c, L.S); break;
      case FORM_SYM: k_assemble_explicit<FORM_SYM><<<nb, kThreads, 0, ctx->stream>>>(g, L.xrows, (int)c, L.S); break;
      default: k_assemble_explicit<FORM_GRAD><<<nb, kThreads, 0, ctx->stream>>>(g, L.xrows, (int)c, L.S); break;
    }
    ST(launched(ctx));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->rl = rl;
  if (fl < 0) return STK_OK;
  // phase program (the V-cycle of op_vcycle / op_uzawa restricted to levels fl..)
  static const int single = getenv("STK_FUSED_SINGLE") ? atoi(getenv("STK_FUSED_SINGLE")) : 1000;
  const int nl = ctx->nlev - fl;
  std::vector<int> m(nl);
  for (int q = 0; q < nl; ++q) {
    const int64_t V = owned_vertices(ctx->lev[fl + q]);
    m[q] = V <= single ? 1 : std::max(1, std::min(ctx->fcluster ? FCL : ctx->fgrid, (int)((V + 255) / 256)));
  }
  const int mc = m[nl - 1] == 1 ? 1 : std::max(1, std::min(ctx->fcluster ? FCL : ctx->fgrid, (ctx->cN + 7) / 8));
  std::vector<FPhase> prog;
  auto add = [&](int op, int lev, int mm, int color = 0, int flip = 0) {
    FPhase P{};
    P.op = (uint8_t)op;
    P.lev = (uint8_t)lev;
    P.color = (uint8_t)color;
    P.flip = (uint8_t)flip;
    P.m = (int16_t)mm;
    prog.push_back(P);
  };
  const int nc = ctx->cfg.ncolors_u;
  auto uzawa = [&](int q) {
    for (int s = 0; s < 2 * nc; ++s) add(FPH_VEL, q, m[q], s < nc ? s : 2 * nc - 1 - s, s & 1);
    add(FPH_P1, q, m[q]);
    add(FPH_P2, q, m[q]);
  };
  add(FPH_ZERO, 0, m[0]);
  for (int q = 0; q + 1 < nl; ++q) {
    const int nu = ctx->cfg.nu_pre + ctx->cfg.nu_inc * (fl + q);
    for (int s = 0; s < nu; ++s) uzawa(q);
    add(FPH_RES, q, m[q]);
    add(FPH_RESTRICT, q, m[q + 1]);
  }
  add(FPH_COARSE, nl - 1, mc);
  for (int q = nl - 2; q >= 0; --q) {
    const int nu = ctx->cfg.nu_post + ctx->cfg.nu_inc * (fl + q);
    add(FPH_PROLONG, q, m[q]);
    for (int s = 0; s < nu; ++s) uzawa(q);
  }
  if ((int)prog.size() > FPH_MAX) return STK_OK;  // too long: per-phase launches
  int gmax = 1;
  for (size_t k = 0; k < prog.size(); ++k) {
    const int next = k + 1 < prog.size() ? prog[k + 1].m : 0;
    prog[k].barM = (int16_t)(next ? std::max<int>(prog[k].m, next) : 0);
    gmax = std::max<int>(gmax, prog[k].m);
  }
  if (!ctx->fprog) CK(cudaMalloc(&ctx->fprog, sizeof(FPhase) * FPH_MAX));
  CK(cudaMemcpy(ctx->fprog, prog.data(), sizeof(FPhase) * prog.size(), cudaMemcpyHostToDevice));
  ctx->fnph = (int)prog.size();
  ctx->fgrid_used = gmax;
  ctx->fl = fl;
  return STK_OK;
}

void drop_graphs(stk_ctx* ctx) {
  if (ctx->coarse_exec) cudaGraphExecDestroy(ctx->coarse_exec);
  ctx->coarse_exec = nullptr;
}

stk_status check(const stk_ctx* ctx, int need_state) {
  if (!ctx) return STK_EINVAL;
  if (ctx->state < need_state) {
    const_cast<stk_ctx*>(ctx)->err = "call order violated (create -> set_viscosity -> assemble)";
    return STK_ESTATE;
  }
  return STK_OK;
}

stk_status check_level(stk_ctx* ctx, int l) {
  if (l < 0 || l >= ctx->nlev) {
    ctx->err = "level out of range";
    return STK_EINVAL;
  }
  return STK_OK;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

stk_status stk_nccl_unique_id(uint8_t id[128]) { return comm_unique_id(id); }

stk_status stk_partition(int32_t n, int32_t n_coarse, int32_t nranks, int32_t rank, int32_t* nlev, int32_t* out) {
  if (!nlev || !out || n < 4 || (n & (n - 1)) != 0 || nranks < 1 || rank < 0 || rank >= nranks) return STK_EINVAL;
  const int nc = n_coarse > 0 ? n_coarse : 4;
  if (nc > n || (nc & (nc - 1)) != 0) return STK_EINVAL;
  std::vector<SlabLevel> part;
  slab_partition(n, nc, nranks, rank, part);
  if (part.size() > 16) return STK_EINVAL;
  *nlev = (int32_t)part.size();
  for (size_t l = 0; l < part.size(); ++l) {
    const SlabLevel& L = part[l];
    const int32_t v[8] = {L.n, L.z0, L.nzl, L.cz0, L.cz1, L.replicated, L.K0, L.K1};
    memcpy(out + 8 * l, v, sizeof(v));
  }
  return STK_OK;
}

namespace {
stk_status create_impl(const stk_config* cfg, const uint8_t* id, stk_loopback* group, stk_ctx** out);
}

stk_status stk_create(const stk_config* cfg, const uint8_t* id, stk_ctx** out) {
  return create_impl(cfg, id, nullptr, out);
}

stk_status stk_loopback_create(int32_t nranks, stk_loopback** out) {
  if (!out || nranks < 1 || nranks > LB_MAXP) return STK_EINVAL;
  stk_loopback* g = new stk_loopback();
  g->P = nranks;
  g->ptr.assign(nranks, nullptr);
  g->aux.assign(nranks, 0);
  if (cudaMalloc(&g->dsum, sizeof(double) * 256) != cudaSuccess) {
    cudaGetLastError();
    delete g;
    return STK_ENOMEM;
  }
  *out = g;
  return STK_OK;
}

stk_status stk_loopback_destroy(stk_loopback* g) {
  if (!g) return STK_EINVAL;
  cudaFree(g->dsum);
  delete g;
  return STK_OK;
}

stk_status stk_create_loopback(const stk_config* cfg, stk_loopback* group, stk_ctx** out) {
  if (!group || !cfg) return STK_EINVAL;
  {
    std::lock_guard<std::mutex> lk(group->m);
    if (!group->stream) group->stream = cfg->stream ? cfg->stream : (void*)1;
    else if (group->stream != (cfg->stream ? cfg->stream : (void*)1)) return STK_EINVAL;  // one stream for all ranks
  }
  return create_impl(cfg, nullptr, group, out);
}

}  // extern "C"

namespace {
stk_status create_impl(const stk_config* cfg, const uint8_t* id, stk_loopback* group, stk_ctx** out) {
  if (!cfg || !out) return STK_EINVAL;
  *out = nullptr;
  const int n = cfg->n;
  if (n < 4 || (n & (n - 1)) != 0) return STK_EINVAL;
  if (cfg->form < 0 || cfg->form > 2) return STK_EINVAL;
  if (cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks) return STK_EINVAL;
  if (cfg->ncolors_u != 2 && cfg->ncolors_u != 4) return STK_EINVAL;
  if (cfg->krylov < 0 || cfg->krylov > 200) return STK_EINVAL;
  if (cfg->coarse_mu < 0 || cfg->coarse_mu > 2) return STK_EINVAL;
  const int nc = cfg->n_coarse > 0 ? cfg->n_coarse : 4;
  if (nc > n || (nc & (nc - 1)) != 0 || nc > 16) return STK_EINVAL;
  bool any_dir = false, slip_axis[3] = {false, false, false};
  for (int f = 0; f < 6; ++f) {
    if (cfg->face[f] != STK_FACE_DIRICHLET0 && cfg->face[f] != STK_FACE_TRACTION && cfg->face[f] != STK_FACE_FREESLIP)
      return STK_EINVAL;
    any_dir |= cfg->face[f] == STK_FACE_DIRICHLET0;
    slip_axis[f / 2] |= cfg->face[f] == STK_FACE_FREESLIP;
  }
  // Korn: |Gamma_D| > 0, or free-slip faces of all three normal directions
  // (u.n = 0 on faces x, y and z excludes the rigid translations and rotations)
  if (!any_dir && !(slip_axis[0] && slip_axis[1] && slip_axis[2])) return STK_EINVAL;
  stk_ctx* ctx = new stk_ctx();
  ctx->cfg = *cfg;
  ctx->cfg.n_coarse = nc;
  if (ctx->cfg.delta <= 0) ctx->cfg.delta = 1.0 / 12.0;
  ctx->stream = (cudaStream_t)cfg->stream;
  // constant tables
  int8_t perm[6][3], corner[8][6], choff[6][8], cht[6][8];
  host_tables(perm, corner, choff, cht);
  auto fail = [&](stk_status s) { *out = ctx; return s; };
  if (cudaMemcpyToSymbol(c_perm, perm, sizeof(perm)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_corner_m, corner, sizeof(corner)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_child_off, choff, sizeof(choff)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_child_t, cht, sizeof(cht)) != cudaSuccess) {
    ctx->err = "cudaMemcpyToSymbol failed (no CUDA device?)";
    return fail(STK_ECUDA);
  }
  // communicator
  stk_status s = ctx->comm.init(ctx, cfg->rank, cfg->nranks, id, group);
  if (s != STK_OK) return fail(s);
  // levels
  for (int m = n; m >= nc; m /= 2) {
    Level L;
    L.n = m;
    L.h = 1.0 / m;
    ctx->lev.push_back(L);
  }
  ctx->nlev = (int)ctx->lev.size();
  std::vector<SlabLevel> part;
  slab_partition(n, nc, cfg->nranks, cfg->rank, part);
  for (int l = 0; l < ctx->nlev; ++l) {
    Level& L = ctx->lev[l];
    L.replicated = part[l].replicated;
    L.z0 = part[l].z0;
    L.nzl = part[l].nzl;
    L.cz0 = part[l].cz0;
    L.cz1 = part[l].cz1;
    L.px = ((L.n + 3 + 15) / 16) * 16;  // ghost column i = -1, vertices 0..n, spare
    L.py = L.px * (L.n + 2);             // ghost row j = -1, rows 0..n
    // planes z0-1 .. z0+nzl (halos included) plus one spare plane: the row kernels
    // gather the Kuhn offset (0,1,1) of a vertex on the top-back edge without bounds
    // checks, i.e. row j = n+1 of the top halo plane = the spare plane's ghost row
    // (0 by the level-vector invariant) -- without it that read left the field
    L.fs = (((int64_t)(L.nzl + 3) * L.py + 31) / 32) * 32;
    L.vlen = 4 * L.fs;
    const size_t ncls = (size_t)(L.cz1 - L.cz0) * L.n * L.n * 6;
    if (cudaMalloc(&L.cls, ncls) != cudaSuccess ||
        cudaMalloc(&L.code, sizeof(uint8_t) * L.fs) != cudaSuccess ||
        cudaMalloc(&L.r, sizeof(double) * L.vlen) != cudaSuccess) {
      ctx->err = "out of device memory (level arrays)";
      return fail(STK_ENOMEM);
    }
    cudaMemset(L.r, 0, sizeof(double) * L.vlen);
    cudaMemset(L.code, CODE_IRREGULAR, L.fs);
    if (l > 0) {
      if (cudaMalloc(&L.emu, sizeof(double2) * ncls) != cudaSuccess) {
        ctx->err = "out of device memory (coarse element coefficients)";
        return fail(STK_ENOMEM);
      }
      if (cudaMalloc(&L.x, sizeof(double) * L.vlen) != cudaSuccess ||
          cudaMalloc(&L.b, sizeof(double) * L.vlen) != cudaSuccess) {
        ctx->err = "out of device memory (MG vectors)";
        return fail(STK_ENOMEM);
      }
      cudaMemset(L.x, 0, sizeof(double) * L.vlen);
      cudaMemset(L.b, 0, sizeof(double) * L.vlen);
    }
  }
  ctx->nparts = 296;
  if (cudaMalloc(&ctx->part, sizeof(double) * 6 * ctx->nparts) != cudaSuccess ||
      cudaMalloc(&ctx->sums, sizeof(double) * 8) != cudaSuccess ||
      cudaMallocHost(&ctx->hsums, sizeof(double) * 8) != cudaSuccess ||
      cudaMalloc(&ctx->cstatus, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&ctx->d_mu, sizeof(double) * 512) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    ctx->err = "allocation failed";
    return fail(STK_ENOMEM);
  }
  *out = ctx;
  return STK_OK;
}
}  // namespace

extern "C" {

stk_status stk_cube_range(const stk_ctx* ctx, int32_t* z0, int32_t* z1) {
  if (!ctx || !z0 || !z1) return STK_EINVAL;
  *z0 = ctx->lev[0].cz0;
  *z1 = ctx->lev[0].cz1;
  return STK_OK;
}

stk_status stk_set_viscosity(stk_ctx* ctx, const uint8_t* elem_class, const double* class_mu,
                             int32_t nclass) {
  ST(check(ctx, 0));
  if (!elem_class || !class_mu || nclass < 1 || nclass > 254) return STK_EINVAL;  // 0xFE, 0xFF reserved
  double mu[256], imu[256];
  for (int q = 0; q < 256; ++q) mu[q] = imu[q] = 1.0;
  for (int q = 0; q < nclass; ++q) {
    if (!(class_mu[q] > 0.0)) {
      ctx->err = "viscosities must be positive";
      return STK_EINVAL;
    }
    mu[q] = class_mu[q];
    imu[q] = 1.0 / class_mu[q];
  }
  ctx->class_mu.assign(class_mu, class_mu + nclass);
  CK(cudaMemcpyAsync(ctx->d_mu, mu, sizeof(mu), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_mu + 256, imu, sizeof(imu), cudaMemcpyHostToDevice, ctx->stream));
  memcpy(ctx->mutab.mu, mu, sizeof(mu));
  memcpy(ctx->mutab.imu, imu, sizeof(imu));
  Level& L = ctx->lev[0];
  const size_t ncls = (size_t)(L.cz1 - L.cz0) * L.n * L.n * 6;
  CK(cudaMemcpyAsync(L.cls, elem_class, ncls, cudaMemcpyHostToDevice, ctx->stream));
  if (!ctx->dcnt) CK(cudaMalloc(&ctx->dcnt, sizeof(unsigned long long) * (ctx->nlev + 1)));
  CK(cudaMemsetAsync(ctx->dcnt, 0, sizeof(unsigned long long), ctx->stream));
  k_count_ge<<<nblocks((int64_t)ncls), kThreads, 0, ctx->stream>>>(L.cls, (int64_t)ncls, nclass, ctx->dcnt);
  ST(launched(ctx));
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->dcnt, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad) {
    ctx->err = "element class >= nclass";
    return STK_EINVAL;
  }
  ctx->state = std::max(ctx->state, 1);
  if (ctx->state > 1) ctx->state = 1;  // re-assemble required
  return STK_OK;
}

stk_status stk_assemble(stk_ctx* ctx) {
  ST(check(ctx, 1));
  // coarse element classes and coefficients (R15), finest to coarsest
  const int P = ctx->cfg.nranks, rank = ctx->cfg.rank;
  for (int l = 1; l < ctx->nlev; ++l) {
    Level& F = ctx->lev[l - 1];
    Level& C = ctx->lev[l];
    const int64_t lay = (int64_t)C.n * C.n * 6;  // tets per cube layer
    auto coarsen = [&](int CK0, int CK1) -> stk_status {
      const int64_t tot = (int64_t)(CK1 - CK0) * lay;
      if (tot <= 0) return STK_OK;
      k_coarsen<<<nblocks(tot), kThreads, 0, ctx->stream>>>(dgrid(ctx, F), dgrid(ctx, C), CK0, CK1, C.cls, C.emu,
                                                            ctx->cfg.coarse_mu == STK_COARSE_MU_HARMONIC);
      return launched(ctx);
    };
    if (C.replicated && !F.replicated) {
      // coarse layer CK derives from fine layers 2CK, 2CK+1: every rank computes the
      // coarse layers of its fine slab, then the layers are gathered on every rank
      const int per = F.n / P;
      ST(coarsen(rank * per / 2, (rank + 1) * per / 2));
      auto rng = [&](int64_t esz) {
        return [=](int q, int64_t& off, int64_t& len) {
          off = (int64_t)(q * per / 2) * lay * esz;
          len = (int64_t)((q + 1) * per / 2 - q * per / 2) * lay * esz;
        };
      };
      ST(ctx->comm.allgather_ranges(ctx, C.cls, rng(1)));
      ST(ctx->comm.allgather_ranges(ctx, (uint8_t*)C.emu, rng(sizeof(double2))));
    } else if (C.replicated || P == 1 || C.cz0 == C.z0) {
      ST(coarsen(C.cz0, C.cz1));
      if (!C.replicated && P > 1) {  // rank 0 of a split level still sends its top layer up
        ST(ctx->comm.shift_up(ctx, C.cls, (C.cz1 - 1 - C.cz0) * lay, lay));
        ST(ctx->comm.shift_up(ctx, (uint8_t*)C.emu, (C.cz1 - 1 - C.cz0) * lay * (int64_t)sizeof(double2),
                              lay * (int64_t)sizeof(double2)));
      }
    } else {
      // split level, rank > 0: the layers of the own fine slab [z0, cz1); the lowest
      // stored layer z0 - 1 (needs fine layer 2 z0 - 2, not stored here) comes from
      // rank - 1, whose top computed layer it is
      ST(coarsen(C.z0, C.cz1));
      ST(ctx->comm.shift_up(ctx, C.cls, (C.cz1 - 1 - C.cz0) * lay, lay));
      ST(ctx->comm.shift_up(ctx, (uint8_t*)C.emu, (C.cz1 - 1 - C.cz0) * lay * (int64_t)sizeof(double2),
                            lay * (int64_t)sizeof(double2)));
    }
  }
  // classification
  if (!ctx->dcnt) CK(cudaMalloc(&ctx->dcnt, sizeof(unsigned long long) * (ctx->nlev + 1)));
  unsigned long long* dcnt = ctx->dcnt;
  CK(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * ctx->nlev, ctx->stream));
  for (int l = 0; l < ctx->nlev; ++l) {
    Level& L = ctx->lev[l];
    k_classify<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), L.code, dcnt + l);
    ST(launched(ctx));
  }
  std::vector<unsigned long long> cnt(ctx->nlev);
  CK(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(unsigned long long) * ctx->nlev, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int l = 0; l < ctx->nlev; ++l) ctx->lev[l].nirr = (int64_t)cnt[l];
  // compact list rows of the tiled levels (the list role of k_stream): the Gamma rows
  // first, then the isoviscous traction-face rows (which also couple within a colour:
  // the repeat pass of the smoother takes both); one explicit stencil each
  for (int l = 0; l < ctx->nlev; ++l) {
    Level& L = ctx->lev[l];
    L.list = nullptr;
    L.Slist = nullptr;
    L.nrl = 0;
    if (L.n < 64) continue;
    unsigned long long* tc = ctx->dcnt + ctx->nlev;
    CK(cudaMemsetAsync(tc, 0, sizeof(unsigned long long), ctx->stream));
    k_count_top<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), tc);
    ST(launched(ctx));
    unsigned long long ntop = 0;
    CK(cudaMemcpyAsync(&ntop, tc, sizeof(ntop), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    L.nrl = L.nirr + (int64_t)ntop;
    if (L.nrl == 0) continue;
    if (!ensure(L.rlist, L.cap_rlist, (size_t)L.nrl) || !ensure(L.Srl, L.cap_Srl, (size_t)EXPL * L.nrl) ||
        !ensure(L.cbuf, L.cap_cbuf, (size_t)3 * L.nrl))
      return STK_ENOMEM;
    CK(cudaMemsetAsync(tc, 0, sizeof(unsigned long long), ctx->stream));
    k_build_list<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), L.rlist, tc, 0);
    ST(launched(ctx));
    CK(cudaMemsetAsync(tc, 0, sizeof(unsigned long long), ctx->stream));
    k_build_list<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), L.rlist + L.nirr, tc, 1);
    ST(launched(ctx));
    const unsigned nbr = nblocks((int64_t)L.nrl * NQ * 4);
    DGrid gl = dgrid(ctx, L);
    switch (ctx->cfg.form) {
      case FORM_MOD: k_assemble_explicit<FORM_MOD><<<nbr, kThreads, 0, ctx->stream>>>(gl, L.rlist, (int)L.nrl, L.Srl); break;
      case FORM_SYM: k_assemble_explicit<FORM_SYM><<<nbr, kThreads, 0, ctx->stream>>>(gl, L.rlist, (int)L.nrl, L.Srl); break;
      default: k_assemble_explicit<FORM_GRAD><<<nbr, kThreads, 0, ctx->stream>>>(gl, L.rlist, (int)L.nrl, L.Srl); break;
    }
    ST(launched(ctx));
    if (L.nirr > 0) {  // the Gamma rows are the head of the repeat list
      L.list = L.rlist;
      L.Slist = L.Srl;
    }
  }
  // constant subdomain stencils for the tiled kernels
  for (int l = 0; l < ctx->nlev; ++l) {
    Level& L = ctx->lev[l];
    if (ctx->kernel_mode == 1 && L.n >= 64 && !L.replicated && !tiled_supported(L.n)) {
      ctx->err = "tiled kernels unavailable (cuTensorMapEncodeTiled not found): no silent fallback";
      return STK_EUNSUP;
    }
    if (L.n >= 64 && !assemble_stencils(ctx->stream)) {
      ctx->err = "constant stencil assembly failed or disagrees with the compile-time stencils";
      return STK_ECUDA;
    }
  }
  Level& L = ctx->lev[ctx->nlev - 1];
  if (ctx->coarse_kind == 1) {
    // the paper's coarse solver: A_sym explicit stencils of every vertex of the level
    if (!L.replicated && ctx->cfg.nranks > 1) {
      ctx->err = "MINRES coarse solver needs the coarsest level held whole by every rank";
      return STK_EUNSUP;
    }
    const int64_t V = owned_vertices(L);
    if (!ensure(ctx->mr_S, ctx->cap_mr_S, (size_t)EXPL * V) || !ensure(ctx->mr_rows, ctx->cap_mr_rows, (size_t)V) ||
        !ensure(ctx->mr_work, ctx->cap_mr_work, (size_t)MR_NVEC * 4 * V))
      return STK_ENOMEM;
    k_iota<<<nblocks(V), kThreads, 0, ctx->stream>>>(ctx->mr_rows, V);
    ST(launched(ctx));
    k_assemble_explicit<FORM_SYM><<<nblocks(V * NQ * 4), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), ctx->mr_rows,
                                                                                        (int)V, ctx->mr_S);
    ST(launched(ctx));
    ctx->cN = ctx->cN1 = 0;
    ST(fused_setup(ctx));
  } else {
  // coarsest level: dense K (+ gauge row), Gauss-Jordan inverse
  std::vector<int32_t> dofs;
  const unsigned dm = dirmask_of(ctx->cfg), sm = slipmask_of(ctx->cfg);
  for (int k = L.z0; k < L.z0 + L.nzl; ++k)
    for (int j = 0; j <= L.n; ++j)
      for (int i = 0; i <= L.n; ++i) {
        const unsigned em = elim_mask(dm, sm, L.n, i, j, k);
        for (int f = 0; f < 4; ++f)
          if (!((em >> f) & 1u)) dofs.push_back((f << 28) | (k << 18) | (j << 9) | i);
      }
  std::sort(dofs.begin(), dofs.end(), [](int32_t a, int32_t b) {
    const int fa = (a >> 28) & 0xF, fb = (b >> 28) & 0xF;
    if (fa != fb) return fa < fb;
    return (a & 0x0FFFFFFF) < (b & 0x0FFFFFFF);
  });
  const bool gauge = !has_traction(ctx->cfg);
  ctx->cN = (int)dofs.size();
  ctx->cN1 = ctx->cN + (gauge ? 1 : 0);
  const int N1 = ctx->cN1;
  if (!ensure(ctx->cdofs, ctx->cap_cdofs, (size_t)ctx->cN) || !ensure(ctx->cK, ctx->cap_cK, (size_t)N1 * N1) ||
      !ensure(ctx->cG, ctx->cap_cG, (size_t)N1 * N1))
    return STK_ENOMEM;
  CK(cudaMemcpyAsync(ctx->cdofs, dofs.data(), sizeof(int32_t) * ctx->cN, cudaMemcpyHostToDevice, ctx->stream));
  DGrid g = dgrid(ctx, L);
  const unsigned nb = nblocks((int64_t)N1 * N1);
  switch (ctx->cfg.form) {
    case FORM_MOD: k_coarse_assemble<FORM_MOD><<<nb, kThreads, 0, ctx->stream>>>(g, ctx->cdofs, ctx->cN, N1, ctx->cK, gauge); break;
    case FORM_SYM: k_coarse_assemble<FORM_SYM><<<nb, kThreads, 0, ctx->stream>>>(g, ctx->cdofs, ctx->cN, N1, ctx->cK, gauge); break;
    default: k_coarse_assemble<FORM_GRAD><<<nb, kThreads, 0, ctx->stream>>>(g, ctx->cdofs, ctx->cN, N1, ctx->cK, gauge); break;
  }
  ST(launched(ctx));
  CK(cudaMemsetAsync(ctx->cstatus, 0, sizeof(int), ctx->stream));
  ST(fused_setup(ctx));  // grid size + barrier words (used by the coarse inverse too)
  static const bool gj_grid = getenv("STK_GJ_GRID") && atoi(getenv("STK_GJ_GRID"));
  const size_t gsm = gj_cluster_smem(N1);
  if (!gj_grid && gsm <= 220 * 1024) {  // one 8-CTA cluster, matrix in distributed shared memory
    CK(cudaFuncSetAttribute(k_gauss_jordan_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
    k_gauss_jordan_cluster<<<GJC, GJC_NT, gsm, ctx->stream>>>(ctx->cK, ctx->cG, N1, ctx->cstatus);
    ST(launched(ctx));
  } else {
    if (!ensure(ctx->cfac, ctx->cap_cfac, (size_t)N1)) return STK_ENOMEM;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(std::min(ctx->fgrid, std::max(1, (N1 * N1 + 255) / 256)));
    lc.blockDim = dim3(256);
    lc.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, k_gauss_jordan_coop, ctx->cK, ctx->cG, ctx->cfac, N1, ctx->cstatus, ctx->fbar));
    ST(launched(ctx));
  }
  }
  ST(fused_assemble(ctx));
  if (ctx->coarse_kind == 0) {
    int hs = 0;
    CK(cudaMemcpyAsync(&hs, ctx->cstatus, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (hs) {
      ctx->err = "coarse-level matrix is singular";
      return STK_ECUDA;
    }
  } else {
    CK(cudaStreamSynchronize(ctx->stream));
  }
  // keep the captured coarse graph when nothing it depends on changed (pointers,
  // list / explicit-row counts, kernel selection); the data behind them is updated
  std::vector<int64_t> sig = {ctx->kernel_mode, ctx->rl, ctx->fl, ctx->row_n, ctx->fuse_n, ctx->cN, ctx->cN1,
                              (int64_t)ctx->cdofs, (int64_t)ctx->cG, (int64_t)ctx->fprog, ctx->fnph,
                              ctx->coarse_kind, ctx->mr_its, ctx->mr_cg, (int64_t)ctx->mr_S, (int64_t)ctx->mr_work};
  for (auto& Lv : ctx->lev)
    for (int64_t v : {(int64_t)Lv.list, Lv.nirr, (int64_t)Lv.Slist, (int64_t)Lv.slot, (int64_t)Lv.S, Lv.nexpl,
                      (int64_t)Lv.rlist, Lv.nrl, (int64_t)Lv.Srl})
      sig.push_back(v);
  for (int q = 0; q < 256; ++q) {  // the row kernels take the class table by value
    int64_t b;
    memcpy(&b, &ctx->mutab.mu[q], 8);
    sig.push_back(b);
  }
  if (sig != ctx->graph_sig) drop_graphs(ctx);
  ctx->graph_sig = sig;
  ctx->state = 2;
  return STK_OK;
}

stk_status stk_layout(const stk_ctx* ctx, int32_t level, stk_layout_t* out) {
  if (!ctx || !out || level < 0 || level >= ctx->nlev) return STK_EINVAL;
  const Level& L = ctx->lev[level];
  out->n = L.n;
  out->nx = out->ny = L.n + 1;
  out->nz_local = L.nzl;
  out->z0 = L.z0;
  out->pitch_x = L.px;
  out->pitch_y = L.py;
  out->field_stride = L.fs;
  out->vec_len = L.vlen;
  out->n_irregular = L.nirr;
  out->n_vertices = owned_vertices(L);
  return STK_OK;
}

stk_status stk_import(stk_ctx* ctx, int32_t level, const double* canon, int32_t where, double* dev) {
  ST(check(ctx, 0));
  ST(check_level(ctx, level));
  Level& L = ctx->lev[level];
  const size_t bytes = sizeof(double) * 4 * owned_vertices(L);
  const double* src = canon;
  double* staging = nullptr;
  if (where == STK_HOST) {
    CK(cudaMallocAsync(&staging, bytes, ctx->stream));
    CK(cudaMemcpyAsync(staging, canon, bytes, cudaMemcpyHostToDevice, ctx->stream));
    src = staging;
  }
  k_pack<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), src, dev, 4);
  stk_status s = launched(ctx);
  if (staging) CK(cudaFreeAsync(staging, ctx->stream));
  if (where == STK_HOST) CK(cudaStreamSynchronize(ctx->stream));
  return s;
}

stk_status stk_p0_apply(stk_ctx* ctx, const double* x, const double* p0, double* y, double* y0, double gamma) {
  ST(check(ctx, 2));
  if (!x || !p0 || !y || !y0 || !(gamma > 0)) return STK_EINVAL;
  if (ctx->cfg.nranks != 1) {
    ctx->err = "stk_p0_apply: one rank only";
    return STK_EUNSUP;
  }
  Level& L = ctx->lev[0];
  const DGrid g = dgrid(ctx, L);
  ST(op_apply(ctx, 0, BLK_A, x, y));  // A u (the velocity block is the P1-P1 scheme's)
  k_p0_bt<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(g, p0, y);
  ST(launched(ctx));
  const int64_t E = (int64_t)6 * L.n * L.n * L.n;
  k_p0_rows<<<nblocks(E), kThreads, 0, ctx->stream>>>(g, x, p0, y0, gamma);
  return launched(ctx);
}

stk_status stk_p0_fluxes(stk_ctx* ctx, const double* x, const double* p0, double* flux, double gamma) {
  ST(check(ctx, 2));
  if (!x || !p0 || !flux || !(gamma > 0)) return STK_EINVAL;
  if (ctx->cfg.nranks != 1) {
    ctx->err = "stk_p0_fluxes: one rank only";
    return STK_EUNSUP;
  }
  Level& L = ctx->lev[0];
  const int64_t E = (int64_t)6 * L.n * L.n * L.n;
  k_p0_fluxes<<<nblocks(E), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), x, p0, flux, gamma);
  return launched(ctx);
}

__global__ void k_fill(double* __restrict__ a, int64_t n, double v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    a[e] = v;
}

// The P1-P0 system K0 (u, p0) = (b_u, b0) by right-preconditioned GMRES(m) (CGS2, as
// op_gmres) over composite vectors [level-0 vector (pressure field kept 0) | 6 n^3 per-tet
// pressures].  Preconditioner (auxiliary space): the P0 residual is shared by the 4
// vertices of each tet (k_p0_to_p1), one V_var cycle of the library's P1-P1 multigrid
// (same velocity space and viscous form) is applied, and the P1 pressure correction is
// averaged per tet (k_p1_to_p0).
stk_status stk_p0_solve(stk_ctx* ctx, const double* bu, const double* b0, double* xu, double* x0, double gamma,
                        double rtol, int32_t max_its, int32_t m, stk_report* rep) {
  ST(check(ctx, 2));
  if (!bu || !b0 || !xu || !x0 || !(gamma > 0) || m < 1 || m + 1 > KRY_MAXV || max_its < 1) return STK_EINVAL;
  if (ctx->cfg.nranks != 1) {
    ctx->err = "stk_p0_solve: one rank only";
    return STK_EUNSUP;
  }
  Level& L = ctx->lev[0];
  const DGrid g = dgrid(ctx, L);
  const int64_t vlen = L.vlen, fs = L.fs, E = (int64_t)6 * L.n * L.n * L.n, clen = vlen + E;
  const size_t cb = sizeof(double) * clen;
  // basis (m+1), Z (m), b, x, r, w, two level vectors, ones(E), partials
  const size_t need = (size_t)clen * (2 * m + 5) + 2 * (size_t)vlen + E + (size_t)kGsBlocks * (KRY_MAXV + 1) + 128;
  if (!ensure(ctx->p0ws, ctx->cap_p0ws, need)) return STK_ENOMEM;
  CK(cudaMemsetAsync(ctx->p0ws, 0, sizeof(double) * need, ctx->stream));
  double* Vb = ctx->p0ws;
  double* Zb = Vb + (size_t)clen * (m + 1);
  double* B = Zb + (size_t)clen * m;
  double* X = B + clen;
  double* R = X + clen;
  double* W = R + clen;
  double* pb = W + clen;
  double* zl = pb + vlen;
  double* ones = zl + vlen;
  double* part = ones + E;
  double* coef = part + (size_t)kGsBlocks * (KRY_MAXV + 1);  // 128 device scalars
  auto V = [&](int q) { return Vb + (size_t)q * clen; };
  auto Zq = [&](int q) { return Zb + (size_t)q * clen; };
  k_fill<<<256, 256, 0, ctx->stream>>>(ones, E, 1.0);
  ST(launched(ctx));
  // composite b, x (level parts without the pressure field)
  CK(cudaMemcpyAsync(B, bu, sizeof(double) * 3 * fs, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(B + vlen, b0, sizeof(double) * E, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(X, xu, sizeof(double) * 3 * fs, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(X + vlen, x0, sizeof(double) * E, cudaMemcpyDeviceToDevice, ctx->stream));
  const unsigned nbv = nblocks(owned_vertices(L)), nbe = nblocks(E);
  auto Kop = [&](const double* in, double* out) -> stk_status {
    ST(op_apply(ctx, 0, BLK_A, in, out));
    k_p0_bt<<<nbv, kThreads, 0, ctx->stream>>>(g, in + vlen, out);
    ST(launched(ctx));
    k_p0_rows<<<nbe, kThreads, 0, ctx->stream>>>(g, in, in + vlen, out + vlen, gamma);
    return launched(ctx);
  };
  auto Minv = [&](const double* in, double* out) -> stk_status {
    CK(cudaMemcpyAsync(pb, in, sizeof(double) * 3 * fs, cudaMemcpyDeviceToDevice, ctx->stream));
    k_p0_to_p1<<<nbv, kThreads, 0, ctx->stream>>>(g, in + vlen, pb + 3 * fs);
    ST(launched(ctx));
    CK(cudaMemsetAsync(zl, 0, sizeof(double) * vlen, ctx->stream));
    ST(op_vcycle(ctx, 0, pb, zl));
    CK(cudaMemcpyAsync(out, zl, sizeof(double) * 3 * fs, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemsetAsync(out + 3 * fs, 0, sizeof(double) * fs, ctx->stream));
    k_p1_to_p0<<<nbe, kThreads, 0, ctx->stream>>>(g, zl + 3 * fs, out + vlen, in + vlen, 0.5);
    return launched(ctx);
  };
  // flat CGS passes over composite vectors (k_gs_pass with the composite length)
  auto gs = [&](int mode, const double* Vp, int nv, double* w, const double* c, double* out, int cnt) -> stk_status {
    switch (mode) {
      case GS_DOTS: k_gs_pass<GS_DOTS, KRY_MAXV><<<kGsBlocks, 256, 0, ctx->stream>>>(Vp, clen, nv, w, c, part); break;
      case GS_UPDATE_DOTS:
        k_gs_pass<GS_UPDATE_DOTS, KRY_MAXV><<<kGsBlocks, 256, 0, ctx->stream>>>(Vp, clen, nv, w, c, part);
        break;
      default: k_gs_pass<GS_UPDATE_NORM, KRY_MAXV><<<kGsBlocks, 256, 0, ctx->stream>>>(Vp, clen, nv, w, c, part);
    }
    ST(launched(ctx));
    k_gs_final<<<1, 64, 0, ctx->stream>>>(part, kGsBlocks, cnt, out);
    return launched(ctx);
  };
  auto host = [&](const double* d, int cnt, double* h) -> stk_status {
    CK(cudaMemcpyAsync(h, d, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return STK_OK;
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, ctx->stream));
  stk_report local{};
  stk_report* Rp = rep ? rep : &local;
  memset(Rp, 0, sizeof(*Rp));
  double nb2 = 0.0, nr2 = 0.0;
  ST(gs(GS_UPDATE_NORM, B, 0, B, nullptr, coef, 1));  // ||b||^2 (no update with nv = 0, slot 0 = w . w)
  ST(host(coef, 1, &nb2));
  const double bnorm = std::sqrt(nb2);
  auto residual = [&]() -> stk_status {  // R = B - K X, returns ||R||^2 in nr2
    ST(Kop(X, R));
    k_axpby_flat<<<kGsBlocks, 256, 0, ctx->stream>>>(clen, 1.0, B, -1.0, R);
    ST(launched(ctx));
    ST(gs(GS_UPDATE_NORM, R, 0, R, nullptr, coef, 1));
    return host(coef, 1, &nr2);
  };
  ST(residual());
  double beta = std::sqrt(nr2), rel = bnorm > 0 ? beta / bnorm : 0.0;
  Rp->res_hist[0] = rel;
  int its = 0;
  std::vector<double> H((m + 1) * m, 0.0), cs(m), sn(m), gv(m + 1), h(m + 1), y(m), hc(3 * (m + 2));
  while (rel > rtol && its < max_its) {
    k_axpby_flat<<<kGsBlocks, 256, 0, ctx->stream>>>(clen, 1.0 / beta, R, 0.0, V(0));
    ST(launched(ctx));
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int jdone = 0;
    for (int j = 0; j < m && its < max_its; ++j) {
      ST(Minv(V(j), Zq(j)));
      ST(Kop(Zq(j), W));
      double* c1 = coef;
      double* c2 = coef + (m + 2);
      double* nw = coef + 2 * (m + 2);
      ST(gs(GS_DOTS, V(0), j + 1, W, nullptr, c1, j + 1));
      ST(gs(GS_UPDATE_DOTS, V(0), j + 1, W, c1, c2, j + 1));
      ST(gs(GS_UPDATE_NORM, V(0), j + 1, W, c2, nw, 1));
      ST(host(coef, 3 * (m + 2), hc.data()));
      for (int q = 0; q <= j; ++q) h[q] = hc[q] + hc[(m + 2) + q];
      h[j + 1] = std::sqrt(std::max(hc[2 * (m + 2)], 0.0));
      if (h[j + 1] > 0) {
        k_axpby_flat<<<kGsBlocks, 256, 0, ctx->stream>>>(clen, 1.0 / h[j + 1], W, 0.0, V(j + 1));
        ST(launched(ctx));
      }
      for (int q = 0; q < j; ++q) {
        const double t = cs[q] * h[q] + sn[q] * h[q + 1];
        h[q + 1] = -sn[q] * h[q] + cs[q] * h[q + 1];
        h[q] = t;
      }
      const double den = std::hypot(h[j], h[j + 1]);
      cs[j] = den > 0 ? h[j] / den : 1.0;
      sn[j] = den > 0 ? h[j + 1] / den : 0.0;
      h[j] = den;
      h[j + 1] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      for (int q = 0; q <= j; ++q) H[q * m + j] = h[q];
      ++its;
      jdone = j + 1;
      rel = bnorm > 0 ? std::fabs(gv[j + 1]) / bnorm : 0.0;
      if (its < 256) Rp->res_hist[its] = rel;
      if (!std::isfinite(rel)) {
        Rp->nan_seen = 1;
        break;
      }
      if (rel <= rtol) break;
    }
    for (int q = jdone - 1; q >= 0; --q) {
      double s = gv[q];
      for (int c = q + 1; c < jdone; ++c) s -= H[q * m + c] * y[c];
      y[q] = s / H[q * m + q];
    }
    for (int q = 0; q < jdone; ++q) {
      k_axpby_flat<<<kGsBlocks, 256, 0, ctx->stream>>>(clen, y[q], Zq(q), 1.0, X);
      ST(launched(ctx));
    }
    ST(residual());
    beta = std::sqrt(nr2);
    rel = bnorm > 0 ? beta / bnorm : 0.0;
    if (its < 256) Rp->res_hist[its] = rel;
    if (Rp->nan_seen) break;
  }
  // the volume-weighted (all tets equal) mean of p0 removed when no face is traction free
  if (!has_traction(ctx->cfg)) {
    k_gs_pass<GS_DOTS, 8><<<kGsBlocks, 256, 0, ctx->stream>>>(ones, E, 1, X + vlen, nullptr, part);
    ST(launched(ctx));
    k_gs_final<<<1, 64, 0, ctx->stream>>>(part, kGsBlocks, 1, coef);
    ST(launched(ctx));
    double sp = 0.0;
    ST(host(coef, 1, &sp));
    k_axpby_flat<<<kGsBlocks, 256, 0, ctx->stream>>>(E, -sp / (double)E, ones, 1.0, X + vlen);
    ST(launched(ctx));
  }
  CK(cudaMemcpyAsync(xu, X, sizeof(double) * 3 * fs, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(x0, X + vlen, sizeof(double) * E, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  Rp->cycles = its;
  Rp->rel_res = rel;
  Rp->t_total_s = ms * 1e-3;
  return rel <= rtol ? STK_OK : STK_ENOCONV;
}

stk_status stk_set_coarse_solver(stk_ctx* ctx, int32_t kind, int32_t minres_its, int32_t cg_its) {
  if (!ctx || kind < 0 || kind > 1 || minres_its < 1 || minres_its > 10000 || cg_its < 0 || cg_its > 10000)
    return STK_EINVAL;
  ctx->coarse_kind = kind;
  ctx->mr_its = minres_its;
  ctx->mr_cg = cg_its;
  if (ctx->state == 2) ctx->state = 1;  // re-assemble before the next solve
  return STK_OK;
}

stk_status stk_zero_eliminated(stk_ctx* ctx, int32_t level, double* dev) {
  ST(check(ctx, 0));
  ST(check_level(ctx, level));
  Level& L = ctx->lev[level];
  k_zero_eliminated<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), dev);
  return launched(ctx);
}

stk_status stk_export(stk_ctx* ctx, int32_t level, const double* dev, double* canon, int32_t where) {
  ST(check(ctx, 0));
  ST(check_level(ctx, level));
  Level& L = ctx->lev[level];
  const size_t bytes = sizeof(double) * 4 * owned_vertices(L);
  double* dst = canon;
  double* staging = nullptr;
  if (where == STK_HOST) {
    CK(cudaMallocAsync(&staging, bytes, ctx->stream));
    dst = staging;
  }
  k_unpack<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(dgrid(ctx, L), dev, dst);
  ST(launched(ctx));
  if (where == STK_HOST) {
    CK(cudaMemcpyAsync(canon, staging, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaFreeAsync(staging, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return STK_OK;
}

stk_status stk_load_vector(stk_ctx* ctx, int32_t kind, const void* f_dev, const double* table,
                           int32_t nftab, double* b_dev) {
  ST(check(ctx, 1));
  Level& L = ctx->lev[0];
  DGrid g = dgrid(ctx, L);
  if (kind == 0) {
    ST(ctx->comm.halo(ctx, L.n, L.z0, L.nzl, L.py, L.fs, (double*)f_dev, 0, 3, L.replicated));
    k_load_nodal<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(g, (const double*)f_dev, b_dev);
    return launched(ctx);
  }
  if (kind == 1) {
    if (!table || nftab < 1 || nftab > 256) return STK_EINVAL;
    double* dt;
    CK(cudaMallocAsync(&dt, sizeof(double) * 3 * nftab, ctx->stream));
    CK(cudaMemcpyAsync(dt, table, sizeof(double) * 3 * nftab, cudaMemcpyHostToDevice, ctx->stream));
    k_load_elem<<<nblocks(owned_vertices(L)), kThreads, 0, ctx->stream>>>(g, (const uint8_t*)f_dev, dt, b_dev);
    stk_status s = launched(ctx);
    CK(cudaFreeAsync(dt, ctx->stream));
    return s;
  }
  return STK_EINVAL;
}

stk_status stk_apply(stk_ctx* ctx, int32_t level, uint32_t blocks, const double* x, double* y) {
  ST(check(ctx, 2));
  ST(check_level(ctx, level));
  return op_apply(ctx, level, blocks & BLK_ALL, x, y);
}

stk_status stk_norms(stk_ctx* ctx, int32_t level, const double* x, double* out) {
  ST(check(ctx, 2));
  ST(check_level(ctx, level));
  ST(op_partials(ctx, level, x, 0));
  CK(cudaMemcpyAsync(ctx->hsums, ctx->sums, sizeof(double) * 6, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int q = 0; q < 4; ++q) out[q] = ctx->hsums[q];
  out[4] = out[0] + out[1] + out[2] + out[3];
  return STK_OK;
}

stk_status stk_residual(stk_ctx* ctx, int32_t level, const double* x, const double* b, double* r,
                        double* norms) {
  ST(check(ctx, 2));
  ST(check_level(ctx, level));
  static const bool dbg_rows = getenv("STK_DBG_ROWS") && atoi(getenv("STK_DBG_ROWS"));
  if (dbg_rows && row_level(ctx, level)) {
    Level& L = ctx->lev[level];
    CK(cudaMemcpyAsync(L.x, x, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(L.b, b, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    ST(op_residual_rows(ctx, level));
    CK(cudaMemcpyAsync(r, L.r, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    ST(op_residual(ctx, level, x, b, r));
  }
  if (norms) return stk_norms(ctx, level, r, norms);
  return STK_OK;
}

stk_status stk_smooth(stk_ctx* ctx, int32_t level, double* x, const double* b, int32_t steps) {
  ST(check(ctx, 2));
  ST(check_level(ctx, level));
  if (level == ctx->nlev - 1 && ctx->nlev > 1) { /* allowed: smoothing on the coarsest grid */ }
  static const bool dbg_rows = getenv("STK_DBG_ROWS") && atoi(getenv("STK_DBG_ROWS"));
  static const int dbg_coarse = getenv("STK_DBG_COARSE") ? atoi(getenv("STK_DBG_COARSE")) : 0;
  if (dbg_coarse && level == ctx->nlev - 1) {  // debug: the coarse solve (1: row kernel, 2: one-CTA kernel)
    Level& L = ctx->lev[level];
    CK(cudaMemcpyAsync(L.b, b, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemsetAsync(L.x, 0, sizeof(double) * L.vlen, ctx->stream));
    if (dbg_coarse == 1) ST(op_coarse_rows(ctx));
    else ST(op_coarse(ctx, L.b, L.x));
    CK(cudaMemcpyAsync(x, L.x, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    return STK_OK;
  }
  if (dbg_rows && row_level(ctx, level)) {  // debug: the V-cycle's row kernels on the caller's vectors
    Level& L = ctx->lev[level];
    CK(cudaMemcpyAsync(L.x, x, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(L.b, b, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    for (int s = 0; s < steps; ++s) ST(op_uzawa_rows(ctx, level));
    CK(cudaMemcpyAsync(x, L.x, sizeof(double) * L.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    return STK_OK;
  }
  for (int s = 0; s < steps; ++s) ST(op_uzawa(ctx, level, x, b));
  return STK_OK;
}

stk_status stk_restrict(stk_ctx* ctx, int32_t fine_level, const double* r_f, double* b_c) {
  ST(check(ctx, 2));
  if (fine_level < 0 || fine_level >= ctx->nlev - 1) return STK_EINVAL;
  static const bool dbg_rows = getenv("STK_DBG_ROWS") && atoi(getenv("STK_DBG_ROWS"));
  if (dbg_rows && row_level(ctx, fine_level) && row_level(ctx, fine_level + 1)) {
    Level& F = ctx->lev[fine_level];
    Level& C = ctx->lev[fine_level + 1];
    CK(cudaMemcpyAsync(F.r, r_f, sizeof(double) * F.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    ST(op_restrict_rows(ctx, fine_level));
    CK(cudaMemcpyAsync(b_c, C.b, sizeof(double) * C.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    return STK_OK;
  }
  return op_restrict(ctx, fine_level, r_f, b_c);
}

stk_status stk_prolong_add(stk_ctx* ctx, int32_t coarse_level, const double* x_c, double* x_f) {
  ST(check(ctx, 2));
  if (coarse_level < 1 || coarse_level >= ctx->nlev) return STK_EINVAL;
  static const bool dbg_rows = getenv("STK_DBG_ROWS") && atoi(getenv("STK_DBG_ROWS"));
  if (dbg_rows && row_level(ctx, coarse_level - 1) && row_level(ctx, coarse_level)) {
    Level& F = ctx->lev[coarse_level - 1];
    Level& C = ctx->lev[coarse_level];
    CK(cudaMemcpyAsync(C.x, x_c, sizeof(double) * C.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(F.x, x_f, sizeof(double) * F.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    ST(op_prolong_rows(ctx, coarse_level));
    CK(cudaMemcpyAsync(x_f, F.x, sizeof(double) * F.vlen, cudaMemcpyDeviceToDevice, ctx->stream));
    return STK_OK;
  }
  return op_prolong_add(ctx, coarse_level, x_c, x_f);
}

stk_status stk_vcycle(stk_ctx* ctx, const double* b, double* x) {
  ST(check(ctx, 2));
  return op_vcycle(ctx, 0, b, x);
}

stk_status stk_gauge(stk_ctx* ctx, int32_t level, double* x) {
  ST(check(ctx, 2));
  ST(check_level(ctx, level));
  return op_gauge(ctx, level, x);
}

stk_status stk_solve(stk_ctx* ctx, const double* b, double* x, double rtol, int32_t max_cycles,
                     stk_report* rep) {
  ST(check(ctx, 2));
  Level& L = ctx->lev[0];
  stk_report local{};
  stk_report* R = rep ? rep : &local;
  memset(R, 0, sizeof(*R));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, ctx->stream));
  ctx->lvl_pool.reset();
  ctx->lvl_timing = ctx->nlev > 1;
  double nb[5];
  ST(stk_norms(ctx, 0, b, nb));
  const double bnorm = std::sqrt(nb[4]);
  double nr[5];
  ST(stk_residual(ctx, 0, x, b, L.r, nr));
  double rel = bnorm > 0 ? std::sqrt(nr[4]) / bnorm : 0.0;
  R->res_hist[0] = rel;
  int cyc = 0;
  stk_status st = STK_OK;
  if (ctx->cfg.krylov > 0) {
    ST(op_gmres(ctx, b, x, rtol, max_cycles, R, bnorm, cyc, rel));
  } else {
    while (rel > rtol && cyc < max_cycles) {
      ST(op_vcycle(ctx, 0, b, x));
      ST(stk_residual(ctx, 0, x, b, L.r, nr));
      ++cyc;
      rel = bnorm > 0 ? std::sqrt(nr[4]) / bnorm : 0.0;
      if (cyc < 256) R->res_hist[cyc] = rel;
      if (!std::isfinite(rel)) {
        R->nan_seen = 1;
        break;
      }
    }
  }
  ctx->lvl_timing = 0;
  ST(op_gauge(ctx, 0, x));
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  double coarse_ms = 0.0;
  for (auto& r : ctx->lvl_pool.recs) {
    float t = 0;
    cudaEventElapsedTime(&t, r.e0, r.e1);
    coarse_ms += t;
  }
  ctx->lvl_pool.reset();
  R->t_level_s[0] = (ms - coarse_ms) * 1e-3;
  R->t_level_s[1] = coarse_ms * 1e-3;
  R->cycles = cyc;
  R->rel_res = rel;
  R->t_total_s = ms * 1e-3;
  const int m = std::min(cyc, 255);
  const int first = std::max(1, m - 5);
  R->rho = (m >= 1 && R->res_hist[first - 1] > 0)
               ? std::pow(R->res_hist[m] / R->res_hist[first - 1], 1.0 / (m - first + 1))
               : 0.0;
  if (!(rel <= rtol)) st = STK_ENOCONV;
  return st;
}

stk_status stk_export_classes(stk_ctx* ctx, int32_t level, uint8_t* cls_host, double* emu_host) {
  ST(check(ctx, 2));
  ST(check_level(ctx, level));
  if (!cls_host) return STK_EINVAL;
  Level& L = ctx->lev[level];
  const size_t ncls = (size_t)(L.cz1 - L.cz0) * L.n * L.n * 6;
  CK(cudaMemcpyAsync(cls_host, L.cls, ncls, cudaMemcpyDeviceToHost, ctx->stream));
  if (emu_host) {
    if (L.emu) {
      CK(cudaMemcpyAsync(emu_host, L.emu, sizeof(double2) * ncls, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      memset(emu_host, 0, sizeof(double2) * ncls);
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return STK_OK;
}

stk_status stk_export_codes(stk_ctx* ctx, int32_t level, uint8_t* code_host) {
  ST(check(ctx, 2));
  ST(check_level(ctx, level));
  if (!code_host) return STK_EINVAL;
  Level& L = ctx->lev[level];
  std::vector<uint8_t> pad((size_t)L.fs);
  CK(cudaMemcpyAsync(pad.data(), L.code, (size_t)L.fs, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int64_t nx = L.n + 1;
  for (int k = 0; k < L.nzl; ++k)
    for (int j = 0; j <= L.n; ++j)
      for (int i = 0; i <= L.n; ++i)
        code_host[((int64_t)k * nx + j) * nx + i] =
            pad[(size_t)((int64_t)(k + 1) * L.py + (int64_t)(j + 1) * L.px + (i + 1))];
  return STK_OK;
}

stk_status stk_set_kernel_mode(stk_ctx* ctx, int32_t mode) {
  if (!ctx || (mode != 0 && mode != 1)) return STK_EINVAL;
  ctx->kernel_mode = mode;
  drop_graphs(ctx);
  if (ctx->state >= 2) ST(fused_assemble(ctx));
  return STK_OK;
}

stk_status stk_set_fuse_n(stk_ctx* ctx, int32_t fuse_n) {
  if (!ctx || fuse_n < 0) return STK_EINVAL;
  ctx->fuse_n = fuse_n;
  drop_graphs(ctx);
  if (ctx->state >= 2) ST(fused_assemble(ctx));
  return STK_OK;
}

int32_t stk_fused_level(const stk_ctx* ctx) { return ctx ? ctx->fl : -1; }

stk_status stk_set_row_n(stk_ctx* ctx, int32_t row_n) {
  if (!ctx || row_n < 0) return STK_EINVAL;
  ctx->row_n = row_n;
  drop_graphs(ctx);
  if (ctx->state >= 2) ST(fused_assemble(ctx));
  return STK_OK;
}

int32_t stk_row_level(const stk_ctx* ctx) { return ctx ? ctx->rl : -1; }

int64_t stk_launch_count(const stk_ctx* ctx) { return ctx ? ctx->launches : 0; }

stk_status stk_profile_enable(stk_ctx* ctx, int32_t on) {
  if (!ctx) return STK_EINVAL;
  if (on < 0 || on > 2) return STK_EINVAL;
  ctx->prof.on = on;
  return STK_OK;
}

stk_status stk_profile_reset(stk_ctx* ctx) {
  if (!ctx) return STK_EINVAL;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->prof.reset();
  return STK_OK;
}

stk_status stk_profile_read(stk_ctx* ctx, int32_t op, int32_t level, int64_t* launches, double* ms) {
  if (!ctx || !launches || !ms) return STK_EINVAL;
  CK(cudaStreamSynchronize(ctx->stream));
  int64_t cnt = 0;
  double tot = 0.0;
  for (auto& r : ctx->prof.recs) {
    if (r.op != op || (level >= 0 && r.level != level)) continue;
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.e0, r.e1));
    tot += t;
    ++cnt;
  }
  *launches = cnt;
  *ms = tot;
  return STK_OK;
}

const char* stk_last_error(const stk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

stk_status stk_destroy(stk_ctx* ctx) {
  if (!ctx) return STK_EINVAL;
  for (auto& L : ctx->lev) {
    cudaFree(L.cls);
    cudaFree(L.emu);
    cudaFree(L.code);
    cudaFree(L.x);
    cudaFree(L.b);
    cudaFree(L.r);
    cudaFree(L.slot);
    cudaFree(L.xrows);
    cudaFree(L.S);
    cudaFree(L.rlist);
    cudaFree(L.Srl);
    cudaFree(L.cbuf);
  }
  cudaFree(ctx->fbar);
  cudaFree(ctx->dcnt);
  cudaFree(ctx->fprog);
  cudaFree(ctx->cfac);
  cudaFree(ctx->cdofs);
  cudaFree(ctx->cK);
  cudaFree(ctx->cG);
  cudaFree(ctx->mr_S);
  cudaFree(ctx->mr_rows);
  cudaFree(ctx->mr_work);
  cudaFree(ctx->cstatus);
  cudaFree(ctx->d_mu);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  drop_graphs(ctx);
  if (ctx->cap) cudaStreamDestroy(ctx->cap);
  cudaFree(ctx->part);
  cudaFree(ctx->sums);
  cudaFreeHost(ctx->hsums);
  ctx->comm.destroy();
  ctx->prof.destroy();
  ctx->lvl_pool.destroy();
  cudaFree(ctx->kbasis);
  cudaFree(ctx->kwork);
  cudaFree(ctx->kz);
  cudaFree(ctx->p0ws);
  cudaFree(ctx->kcoef);
  cudaFree(ctx->kpart);
  delete ctx;
  return STK_OK;
}

}  // extern "C"
